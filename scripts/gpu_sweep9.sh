python -m pytest tests/test_gpu_parity.py -q -x -k "variants_bitwise" -p no:cacheprovider 2>&1 | tail -1
FHWT_TUNING=1 FHWT_SYN_DYN=1 FHWT_SYN_DYN_GROUPS=4 FHWT_ANA_DYN_GROUPS=4 python -m pytest tests/test_gpu_parity.py -q -x -k "variants_bitwise" -p no:cacheprovider 2>&1 | tail -1
REPS=2 WL=c4 bash tools/bench_ab.sh "" "FHWT_SYN_DYN=1" "FHWT_SYN_DYN=1 FHWT_SYN_DYN_GROUPS=8" "FHWT_SYN_DYN=1 FHWT_SYN_DYN_GROUPS=64" "FHWT_ANA_DYN_GROUPS=2" "FHWT_ANA_DYN_GROUPS=8" > gpurun_out/sweep9_c4.jsonl
cat gpurun_out/sweep9_c4.jsonl
