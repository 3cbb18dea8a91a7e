python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "warp_private_synthesis" > gpurun_out/k4b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/k4b_pytest.log; tail -3 gpurun_out/k4b_pytest.log
export FHWT_TUNING=1
ROUNDS=6 python tools/cmp_variants.py 5 'SYN:' 'SYN:FHWT_SYN_MODE=7' 'SYN:FHWT_SYN_MODE=7,FHWT_SYN_STAGES=3' 'ANA:' > gpurun_out/k4b.jsonl 2>gpurun_out/k4b.err; cat gpurun_out/k4b.jsonl; tail -3 gpurun_out/k4b.err
BATCH=1 SIZE=32768 ROUNDS=4 python tools/cmp_variants.py 8 'SYN:' 'SYN:FHWT_SYN_MODE=7' 'SYN:FHWT_SYN_MODE=7,FHWT_SYN_STAGES=3' > gpurun_out/k4b_c5.jsonl 2>>gpurun_out/k4b.err; cat gpurun_out/k4b_c5.jsonl
