python -m pytest tests/test_gpu_parity.py -q -x -k "variants_bitwise or global_order or tile_counter" -p no:cacheprovider 2>&1 | tail -1
P=paper_1002_2184_b200
for wl in c4 c5; do
REPS=2 WL=$wl bash tools/bench_ab.sh "" "FHWT_LIB=$P/libfhwt_anu.so" > gpurun_out/sweep25_$wl.jsonl
cat gpurun_out/sweep25_$wl.jsonl
done
