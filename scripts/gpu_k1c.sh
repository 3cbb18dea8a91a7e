python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "warp_specialised" > gpurun_out/k1c_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/k1c_pytest.log; tail -3 gpurun_out/k1c_pytest.log
export FHWT_TUNING=1
ROUNDS=8 python tools/cmp_variants.py 5 'ANA:' 'ANA:FHWT_ANA_FUSED=7' 'ANA:FHWT_ANA_FUSED=7,FHWT_ANA_STAGES=3' 'MB:tma' > gpurun_out/k1c.jsonl 2>gpurun_out/k1c.err; cat gpurun_out/k1c.jsonl; tail -3 gpurun_out/k1c.err
BATCH=1 SIZE=32768 ROUNDS=6 python tools/cmp_variants.py 8 'ANA:' 'ANA:FHWT_ANA_FUSED=7' 'ANA:FHWT_ANA_FUSED=7,FHWT_ANA_STAGES=3' > gpurun_out/k1c_c5.jsonl 2>>gpurun_out/k1c.err; cat gpurun_out/k1c_c5.jsonl
