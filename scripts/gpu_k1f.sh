python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "warp_specialised and 11" > gpurun_out/k1f_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/k1f_pytest.log; tail -3 gpurun_out/k1f_pytest.log
export FHWT_TUNING=1
ROUNDS=6 python tools/cmp_variants.py 5 'ANA:' 'ANA:FHWT_ANA_FUSED=11' 'ANA:FHWT_ANA_FUSED=11,FHWT_ANA_CTAS_PER_SM=2' 'MB:ldg' 'MB:tma' > gpurun_out/k1f.jsonl 2>gpurun_out/k1f.err; cat gpurun_out/k1f.jsonl; tail -3 gpurun_out/k1f.err
BATCH=1 SIZE=32768 ROUNDS=4 python tools/cmp_variants.py 8 'ANA:' 'ANA:FHWT_ANA_FUSED=11' > gpurun_out/k1f_c5.jsonl 2>>gpurun_out/k1f.err; cat gpurun_out/k1f_c5.jsonl
