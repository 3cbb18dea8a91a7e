export FHWT_TUNING=1
ROUNDS=8 python tools/cmp_variants.py 5 'ANA:' 'ANA:FHWT_ANA_FUSED=11' 'ANA:FHWT_ANA_FUSED=11,FHWT_ANA_LDG=1' 'ANA:FHWT_ANA_FUSED=11,FHWT_ANA_LDG=2' 'MB:ldg' > gpurun_out/k1g.jsonl 2>gpurun_out/k1g.err; cat gpurun_out/k1g.jsonl; tail -3 gpurun_out/k1g.err
BATCH=1 SIZE=32768 ROUNDS=4 python tools/cmp_variants.py 8 'ANA:' 'ANA:FHWT_ANA_FUSED=11' 'ANA:FHWT_ANA_FUSED=11,FHWT_ANA_LDG=1' 'ANA:FHWT_ANA_FUSED=11,FHWT_ANA_LDG=2' > gpurun_out/k1g_c5.jsonl 2>>gpurun_out/k1g.err; cat gpurun_out/k1g_c5.jsonl
BATCH=1 SIZE=32768 ROUNDS=4 python tools/cmp_variants.py 5 'ANA:' 'ANA:FHWT_ANA_FUSED=11' 'ANA:FHWT_ANA_FUSED=11,FHWT_ANA_LDG=1' > gpurun_out/k1g_c5L5.jsonl 2>>gpurun_out/k1g.err; cat gpurun_out/k1g_c5L5.jsonl
