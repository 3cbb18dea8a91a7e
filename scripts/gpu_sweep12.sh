python -m pytest tests/test_gpu_parity.py -q -x -k "variants_bitwise" -p no:cacheprovider 2>&1 | tail -1
REPS=2 WL=c4 bash tools/bench_ab.sh "" "FHWT_SYN_L1_BOXROWS=8" "FHWT_SYN_L1_BOXROWS=4" "FHWT_SYN_L1_BOXROWS=2" "FHWT_SYN_DYN=1 FHWT_SYN_L1_BOXROWS=8" > gpurun_out/sweep12_c4.jsonl
cat gpurun_out/sweep12_c4.jsonl
