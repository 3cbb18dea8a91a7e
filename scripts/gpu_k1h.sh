export FHWT_TUNING=1
SLEEP=0.4 ROUNDS=12 python tools/cmp_variants.py 5 'ANA:' 'ANA:FHWT_ANA_FUSED=11' 'SYN:' > gpurun_out/k1h.jsonl 2>gpurun_out/k1h.err; cat gpurun_out/k1h.jsonl; tail -3 gpurun_out/k1h.err
SLEEP=0.4 BATCH=1 SIZE=32768 ROUNDS=8 python tools/cmp_variants.py 8 'ANA:' 'ANA:FHWT_ANA_FUSED=11' 'SYN:' > gpurun_out/k1h_c5.jsonl 2>>gpurun_out/k1h.err; cat gpurun_out/k1h_c5.jsonl
