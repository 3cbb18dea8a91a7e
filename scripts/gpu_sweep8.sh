python -m pytest tests/test_gpu_parity.py -q -x -k "variants_bitwise" -p no:cacheprovider 2>&1 | tail -1
for wl in c4 c5; do
REPS=2 WL=$wl bash tools/bench_ab.sh "" "FHWT_SYN_DYN=0" > gpurun_out/sweep8_$wl.jsonl
cat gpurun_out/sweep8_$wl.jsonl
done
