python -m pytest tests/test_gpu_parity.py -q -x -k "tile_counter_workspace or variants_bitwise" -p no:cacheprovider 2>&1 | tail -1
P=paper_1002_2184_b200
REPS=2 WL=c4 bash tools/bench_ab.sh "" "FHWT_LIB=$P/libfhwt_ncmp.so" "FHWT_LIB=$P/libfhwt_ncc.so" "FHWT_LIB=$P/libfhwt_nc.so" > gpurun_out/sweep19_c4.jsonl
cat gpurun_out/sweep19_c4.jsonl
