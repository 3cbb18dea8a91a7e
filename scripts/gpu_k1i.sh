export FHWT_TUNING=1
SLEEP=0.4 ROUNDS=10 python tools/cmp_variants.py 5 'ANA:' 'ANA:FHWT_ANA_FUSED=10,FHWT_ANA_LSU_ROWS=0' 'ANA:FHWT_ANA_FUSED=10,FHWT_ANA_LSU_ROWS=0,FHWT_ANA_MINB=3' 'ANA:FHWT_ANA_FUSED=10,FHWT_ANA_LSU_ROWS=0,FHWT_ANA_MINB=3,FHWT_ANA_STAGES=3' 'ANA:FHWT_ANA_FUSED=11' > gpurun_out/k1i.jsonl 2>gpurun_out/k1i.err; cat gpurun_out/k1i.jsonl; tail -3 gpurun_out/k1i.err
SLEEP=0.4 BATCH=1 SIZE=32768 ROUNDS=6 python tools/cmp_variants.py 8 'ANA:' 'ANA:FHWT_ANA_FUSED=10,FHWT_ANA_LSU_ROWS=0,FHWT_ANA_MINB=3' > gpurun_out/k1i_c5.jsonl 2>>gpurun_out/k1i.err; cat gpurun_out/k1i_c5.jsonl
