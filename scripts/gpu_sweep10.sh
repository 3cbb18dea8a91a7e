REPS=2 WL=c4 bash tools/bench_ab.sh "" "FHWT_SYN_STAGES=3" "FHWT_SYN_DYN=1 FHWT_SYN_STAGES=3" "FHWT_SYN_MODE=2" "FHWT_SYN_MODE=7" "FHWT_SYN_ROWBOX_MIN=512" "FHWT_SYN_TC=512" "FHWT_CTAS_PER_SM=1 FHWT_SYN_STAGES=4" > gpurun_out/sweep10_c4.jsonl
cat gpurun_out/sweep10_c4.jsonl
