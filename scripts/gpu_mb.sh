export FHWT_TUNING=1
ROUNDS=5 python tools/cmp_variants.py 5 'ANA:' 'MB:tma/1/2' 'MB:tma/2/2' 'MB:tma/4/2' 'MB:tma/8/2' 'MB:tma/32/2' 'MB:tma/1/3' 'MB:tma/2/3' 'COPY:' > gpurun_out/mb.jsonl 2>gpurun_out/mb.err; cat gpurun_out/mb.jsonl; tail -3 gpurun_out/mb.err
