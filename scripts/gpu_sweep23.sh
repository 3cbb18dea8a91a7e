python -m pytest tests/test_gpu_parity.py -q -x -k "variants_bitwise or global_order" -p no:cacheprovider 2>&1 | tail -1
FHWT_TUNING=1 FHWT_ANA_DYN_SC=8 FHWT_SYN_DYN_SC=8 python -m pytest tests/test_gpu_parity.py -q -x -k "global_order or c5_reduced or c4_reduced" -p no:cacheprovider 2>&1 | tail -1
REPS=2 WL=c5 bash tools/bench_ab.sh "" "FHWT_ANA_DYN_SC=8" "FHWT_ANA_DYN_SC=32" "FHWT_ANA_DYN_SC=8 FHWT_SYN_DYN_SC=8" > gpurun_out/sweep23_c5.jsonl; cat gpurun_out/sweep23_c5.jsonl
REPS=1 WL=c4 bash tools/bench_ab.sh "" > gpurun_out/sweep23_c4.jsonl; cat gpurun_out/sweep23_c4.jsonl
