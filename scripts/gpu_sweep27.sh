FHWT_TUNING=1 FHWT_ANA_ROWBOXES=0 python -m pytest tests/test_gpu_parity.py -q -x -k "global_order or c4_reduced or c5_reduced" -p no:cacheprovider 2>&1 | tail -1
for wl in c4 c5; do
REPS=2 WL=$wl bash tools/bench_ab.sh "" "FHWT_ANA_ROWBOXES=0" > gpurun_out/sweep27_$wl.jsonl
cat gpurun_out/sweep27_$wl.jsonl
done
