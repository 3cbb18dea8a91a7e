for wl in c4 c5; do
REPS=2 WL=$wl bash tools/bench_ab.sh "" "FHWT_SYN_PROD=2 FHWT_SYN_STAGES=3" "FHWT_ANA_STAGES=3" "FHWT_ANA_STAGES=3 FHWT_SYN_PROD=2 FHWT_SYN_STAGES=3" "FHWT_SYN_PROD=2 FHWT_SYN_STAGES=3 FHWT_SYN_DYN_GROUPS=2" > gpurun_out/sweep14_$wl.jsonl
cat gpurun_out/sweep14_$wl.jsonl
done
