# FUSED=11 register-load analysis variants vs the TMA default: cmp_variants (c4, c5) and the bench line
export FHWT_TUNING=1
python -m pytest tests/test_gpu_parity.py -q -x -k "warp_specialised_analysis_bitwise or variants_bitwise" -p no:cacheprovider 2>&1 | tail -1
for v in 3 4; do FHWT_ANA_FUSED=11 FHWT_ANA_LDG=$v FHWT_DEBUG_LAUNCH=1 python -c "
import torch, paper_1002_2184_b200 as f
x=torch.rand(4,512,2048,device='cuda'); r=f.analyze_2d(x,5)
import os; os.environ['FHWT_ANA_FUSED']='1'; q=f.analyze_2d(x,5); torch.cuda.synchronize(); print('ldg$v bitwise', torch.equal(r,q))
x=torch.rand(1,2048,4096,device='cuda'); r=f.analyze_2d(x,8)
os.environ['FHWT_ANA_FUSED']='11'; q=f.analyze_2d(x,8); torch.cuda.synchronize(); print('ldg$v L8 bitwise', torch.equal(r,q))
" 2>&1 | grep -v "^\[fhwt\] syn"; done
ROUNDS=8 python tools/cmp_variants.py 5 'ANA:' 'ANA:FHWT_ANA_L2HINT=0' 'ANA:FHWT_ANA_FUSED=11' 'ANA:FHWT_ANA_FUSED=11,FHWT_ANA_LDG=3' 'ANA:FHWT_ANA_FUSED=11,FHWT_ANA_LDG=4' 'SYN:' 'COPY:' > gpurun_out/ldg_c4.jsonl 2>gpurun_out/ldg.err; cat gpurun_out/ldg_c4.jsonl; tail -3 gpurun_out/ldg.err
BATCH=1 SIZE=32768 ROUNDS=6 python tools/cmp_variants.py 8 'ANA:' 'ANA:FHWT_ANA_L2HINT=0' 'ANA:FHWT_ANA_FUSED=11' 'ANA:FHWT_ANA_FUSED=11,FHWT_ANA_LDG=3' 'ANA:FHWT_ANA_FUSED=11,FHWT_ANA_LDG=4' 'COPY:' > gpurun_out/ldg_c5.jsonl 2>>gpurun_out/ldg.err; cat gpurun_out/ldg_c5.jsonl
B="python bench.py --steps 20 --warmup 5 --no-breakdown --no-direct --sustained 0 --no-e2e --no-cpu-baseline --no-t1"
for i in 1 2 3; do
  for cfg in "" "FHWT_ANA_L2HINT=0" "FHWT_ANA_FUSED=11" "FHWT_ANA_FUSED=11 FHWT_ANA_LDG=3"; do
    env $cfg $B 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(json.dumps({'cfg': '$cfg', 'value': round(d['value']), 'ana': round(d['kernels']['analysis_gbs']), 'syn': round(d['kernels']['synthesis_gbs']), 'clk': d['clocks'].get('sm_mhz')}))"
  done
done
