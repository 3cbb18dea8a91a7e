python -m pytest tests/test_gpu_parity.py -q -x -k "variants_bitwise" -p no:cacheprovider 2>&1 | tail -1
FHWT_TUNING=1 FHWT_DEBUG_LAUNCH=1 python -c "
import torch, paper_1002_2184_b200 as f, os
for L,shape in ((5,(256,2048,2048)),(8,(1,32768,32768))):
    x=torch.rand(*shape,device='cuda'); a=f.analyze_2d(x,L); r=f.synthesize_2d(a,L)
    os.environ['FHWT_ANA_DYN']='0'; os.environ['FHWT_SYN_DYN']='0'; a2=f.analyze_2d(x,L); r2=f.synthesize_2d(a2,L)
    del os.environ['FHWT_ANA_DYN'], os.environ['FHWT_SYN_DYN']
    torch.cuda.synchronize(); print('dyn full-size bitwise L',L, torch.equal(a,a2), torch.equal(r,r2)); del x,a,a2,r,r2
" 2>&1 | grep -v "^\[fhwt\] ana2d fused 1 tile\|syn2d mode 3"
for wl in c4 c5; do
REPS=2 WL=$wl bash tools/bench_ab.sh "" "FHWT_SYN_DYN=0" "FHWT_ANA_DYN=0 FHWT_SYN_DYN=0" > gpurun_out/sweep7_$wl.jsonl
cat gpurun_out/sweep7_$wl.jsonl
done
python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
