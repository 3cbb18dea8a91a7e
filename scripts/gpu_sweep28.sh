FHWT_TUNING=1 FHWT_LIB=paper_1002_2184_b200/libfhwt_v4.so python -m pytest tests/test_gpu_parity.py -q -x -k "global_order or c4_reduced or c5_reduced or variants_bitwise" -p no:cacheprovider 2>&1 | tail -1
for wl in c4 c5; do
REPS=2 WL=$wl bash tools/bench_ab.sh "" "FHWT_LIB=paper_1002_2184_b200/libfhwt_v4.so" > gpurun_out/sweep28_$wl.jsonl
cat gpurun_out/sweep28_$wl.jsonl
done
