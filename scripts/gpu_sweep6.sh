python -m pytest tests/test_gpu_parity.py -q -x -k "variants_bitwise" -p no:cacheprovider 2>&1 | tail -1
FHWT_TUNING=1 FHWT_ANA_DYN=1 python -c "
import torch, paper_1002_2184_b200 as f, os
for L,shape in ((5,(256,2048,2048)),(8,(1,32768,32768))):
    x=torch.rand(*shape,device='cuda'); a=f.analyze_2d(x,L); a2=f.analyze_2d(x,L)
    os.environ['FHWT_ANA_DYN']='0'; r=f.analyze_2d(x,L); os.environ['FHWT_ANA_DYN']='1'
    torch.cuda.synchronize(); print('dyn full-size bitwise L',L, torch.equal(a,r), torch.equal(a2,r)); del x,a,a2,r
"
for wl in c4 c5; do
REPS=2 WL=$wl bash tools/bench_ab.sh "" "FHWT_ANA_DYN=1" "FHWT_ANA_LEAN=0" > gpurun_out/sweep6_$wl.jsonl
cat gpurun_out/sweep6_$wl.jsonl
done
