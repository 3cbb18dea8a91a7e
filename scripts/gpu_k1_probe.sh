export FHWT_TUNING=1
ROUNDS=4 python tools/offset_probe.py 0 4 64 1024 4096 16384 > gpurun_out/offset_probe.jsonl 2>gpurun_out/offset_probe.err; cat gpurun_out/offset_probe.jsonl; tail -2 gpurun_out/offset_probe.err
ROUNDS=6 python tools/cmp_variants.py 5 'ANA:' 'ANA:FHWT_ANA_FUSED=13' 'ANA:FHWT_ANA_L2HINT=0' 'ANA:FHWT_ANA_FUSED=11' 'COPY:' > gpurun_out/k1p.jsonl 2>gpurun_out/k1p.err; cat gpurun_out/k1p.jsonl; tail -3 gpurun_out/k1p.err
