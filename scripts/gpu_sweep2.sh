python -m pytest tests/test_gpu_parity.py -q -x -k "variants_bitwise" -p no:cacheprovider 2>&1 | tail -1
for wl in c4 c5; do
REPS=2 WL=$wl bash tools/bench_ab.sh "FHWT_ANA_L2HINT=0 FHWT_SYN_L2MODE=1" "FHWT_ANA_L2HINT=0 FHWT_SYN_L2MODE=2" "FHWT_ANA_L2HINT=0 FHWT_SYN_L2MODE=3" > gpurun_out/sweep2_$wl.jsonl
cat gpurun_out/sweep2_$wl.jsonl
done
