export FHWT_TUNING=1
ROUNDS=6 python tools/cmp_variants.py 5 'ANA:' 'ANA:FHWT_ANA_FUSED=7' 'ANA:FHWT_ANA_FUSED=7,FHWT_ANA_POLL=1' 'ANA:FHWT_ANA_FUSED=8,FHWT_ANA_POLL=1' 'MB:tma' > gpurun_out/k1d.jsonl 2>gpurun_out/k1d.err; cat gpurun_out/k1d.jsonl; tail -3 gpurun_out/k1d.err
