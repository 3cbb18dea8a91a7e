# K1 FUSED=12 (refill off the critical path, one CTA barrier per tile) and multi-warp TMA issue
export FHWT_TUNING=1
python -m pytest tests/test_gpu_parity.py -q -x -k "variants_bitwise" -p no:cacheprovider 2>&1 | tail -2
ROUNDS=6 python tools/cmp_variants.py 5 'ANA:' 'ANA:FHWT_ANA_FUSED=12' 'ANA:FHWT_ANA_FUSED=12,FHWT_ANA_STAGES=3' 'MB:tma/1/2' 'MB:tma/1/2/2' 'MB:tma/1/2/4' 'MB:tma/1/3/2' 'COPY:' > gpurun_out/k1f12.jsonl 2>gpurun_out/k1f12.err; cat gpurun_out/k1f12.jsonl; tail -3 gpurun_out/k1f12.err
BATCH=1 SIZE=32768 ROUNDS=4 python tools/cmp_variants.py 8 'ANA:' 'ANA:FHWT_ANA_FUSED=12' > gpurun_out/k1f12_c5.jsonl 2>>gpurun_out/k1f12.err; cat gpurun_out/k1f12_c5.jsonl
