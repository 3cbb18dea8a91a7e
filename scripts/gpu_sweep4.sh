python -m pytest tests/test_gpu_parity.py -q -x -k "variants_bitwise" -p no:cacheprovider 2>&1 | tail -1
REPS=2 WL=c4 bash tools/bench_ab.sh "" "FHWT_ANA_FUSED=9" "FHWT_ANA_FUSED=13" "FHWT_LIB=paper_1002_2184_b200/libfhwt_u32.so" > gpurun_out/sweep4_c4.jsonl
cat gpurun_out/sweep4_c4.jsonl
