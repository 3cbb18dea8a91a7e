python -m pytest tests/test_gpu_parity.py -q -x -k "tile_counter_workspace or variants_bitwise" -p no:cacheprovider 2>&1 | tail -1
for wl in c4 c5; do
REPS=2 WL=$wl bash tools/bench_ab.sh "" "FHWT_SYN_PROD=1" > gpurun_out/sweep21_$wl.jsonl
cat gpurun_out/sweep21_$wl.jsonl
done
