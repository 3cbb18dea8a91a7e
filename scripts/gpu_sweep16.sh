FHWT_TUNING=1 FHWT_DEBUG_LAUNCH=1 FHWT_SYN_TC=512 FHWT_SYN_ROWBOX_MIN=65536 python -c "
import torch, paper_1002_2184_b200 as f
x=torch.rand(8,2048,2048,device='cuda'); c=f.analyze_2d(x,5); r=f.synthesize_2d(c,5); torch.cuda.synchronize(); print('tc512 rt', float((r-x).abs().max()))" 2>&1 | grep -v ana2d
REPS=2 WL=c4 bash tools/bench_ab.sh "" "FHWT_SYN_TC=512 FHWT_SYN_ROWBOX_MIN=65536" "FHWT_SYN_TC=512 FHWT_SYN_ROWBOX_MIN=65536 FHWT_SYN_STAGES=2" "FHWT_SYN_TC=512 FHWT_SYN_ROWBOX_MIN=65536 FHWT_SYN_PROD=0" > gpurun_out/sweep16_c4.jsonl
cat gpurun_out/sweep16_c4.jsonl
