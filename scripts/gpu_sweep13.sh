python -m pytest tests/test_gpu_parity.py -q -x -k "variants_bitwise" -p no:cacheprovider 2>&1 | tail -1
FHWT_TUNING=1 FHWT_SYN_PROD=2 python -m pytest tests/test_gpu_parity.py -q -x -k "c5_reduced or c4_reduced" -p no:cacheprovider 2>&1 | tail -1
REPS=2 WL=c4 bash tools/bench_ab.sh "" "FHWT_SYN_PROD=1" "FHWT_SYN_PROD=2" "FHWT_SYN_PROD=1 FHWT_SYN_STAGES=3" "FHWT_SYN_PROD=2 FHWT_SYN_STAGES=3" > gpurun_out/sweep13_c4.jsonl
cat gpurun_out/sweep13_c4.jsonl
