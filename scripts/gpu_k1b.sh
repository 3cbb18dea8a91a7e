export FHWT_TUNING=1
ROUNDS=6 python tools/cmp_variants.py 5 'ANA:' 'ANA:FHWT_ANA_FUSED=9' 'MB:tma' > gpurun_out/k1b.jsonl 2>gpurun_out/k1b.err; cat gpurun_out/k1b.jsonl; tail -3 gpurun_out/k1b.err
BATCH=1 SIZE=32768 ROUNDS=4 python tools/cmp_variants.py 8 'ANA:' 'ANA:FHWT_ANA_FUSED=9' > gpurun_out/k1b_c5.jsonl 2>>gpurun_out/k1b.err; cat gpurun_out/k1b_c5.jsonl
