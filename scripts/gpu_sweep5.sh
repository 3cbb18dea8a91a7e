python -m pytest tests/test_gpu_parity.py -q -x -k "variants_bitwise" -p no:cacheprovider 2>&1 | tail -1
FHWT_TUNING=1 FHWT_DEBUG_LAUNCH=1 python -c "
import torch, paper_1002_2184_b200 as f
x=torch.rand(2,2048,2048,device='cuda'); f.analyze_2d(x,5); x=torch.rand(1,2048,4096,device='cuda'); f.analyze_2d(x,8); torch.cuda.synchronize()" 2>&1 | grep ana2d
for wl in c4 c5; do
REPS=2 WL=$wl bash tools/bench_ab.sh "" "FHWT_ANA_LEAN=0" "FHWT_LIB=paper_1002_2184_b200/libfhwt_leanu32.so" "FHWT_ANA_FUSED=9" > gpurun_out/sweep5_$wl.jsonl
cat gpurun_out/sweep5_$wl.jsonl
done
