python -m pytest tests/test_gpu_parity.py -q -x -k "variants_bitwise or warp_specialised or warp_private" -p no:cacheprovider 2>&1 | tail -1
REPS=2 WL=c4 bash tools/bench_ab.sh "" "FHWT_ANA_FUSED=3" "FHWT_ANA_FUSED=8" "FHWT_ANA_FUSED=0" "FHWT_ANA_FUSED=11" \
  "FHWT_SYN_MODE=7" "FHWT_SYN_MODE=2" "FHWT_SYN_ROWBOX_MIN=512" "FHWT_SYN_TC=512" "FHWT_ANA_CTAS_PER_SM=1 FHWT_ANA_STAGES=4" > gpurun_out/sweep3_c4.jsonl
cat gpurun_out/sweep3_c4.jsonl
