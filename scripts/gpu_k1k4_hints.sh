# L2 policy / promotion / load-path variants of K1 and K4, rotated order, c4 and c5
export FHWT_TUNING=1
python -m pytest tests/test_gpu_parity.py -q -x -k "variants_bitwise" -p no:cacheprovider 2>&1 | tail -1
ROUNDS=8 python tools/cmp_variants.py 5 'ANA:' 'ANA:FHWT_ANA_L2HINT=0' 'ANA:FHWT_ANA_L2HINT=2' 'ANA:FHWT_ANA_FUSED=11' 'ANA:FHWT_ANA_FUSED=11,FHWT_ANA_LDG=1' 'ANA:FHWT_TMA_L2PROMO=0' 'ANA:FHWT_TMA_L2PROMO=2' 'SYN:' 'SYN:FHWT_SYN_L2MODE=1' 'SYN:FHWT_SYN_L2MODE=2' 'SYN:FHWT_TMA_L2PROMO=0' 'SYN:FHWT_TMA_L2PROMO=2' 'COPY:' > gpurun_out/hints_c4.jsonl 2>gpurun_out/hints.err; cat gpurun_out/hints_c4.jsonl; tail -3 gpurun_out/hints.err
BATCH=1 SIZE=32768 ROUNDS=6 python tools/cmp_variants.py 8 'ANA:' 'ANA:FHWT_ANA_L2HINT=0' 'ANA:FHWT_ANA_L2HINT=2' 'ANA:FHWT_ANA_FUSED=11' 'ANA:FHWT_TMA_L2PROMO=0' 'SYN:' 'SYN:FHWT_SYN_L2MODE=1' 'SYN:FHWT_TMA_L2PROMO=0' 'COPY:' > gpurun_out/hints_c5.jsonl 2>>gpurun_out/hints.err; cat gpurun_out/hints_c5.jsonl
