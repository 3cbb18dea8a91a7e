# K1 variant check: bitwise tests of the warp-specialised analysis, then interleaved A/B timing
python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "warp_specialised or variants_bitwise" > gpurun_out/k1_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/k1_pytest.log; tail -3 gpurun_out/k1_pytest.log
export FHWT_TUNING=1
ROUNDS=6 python tools/cmp_variants.py 5 'ANA:' 'ANA:FHWT_ANA_FUSED=8' 'ANA:FHWT_ANA_FUSED=8,FHWT_ANA_STAGES=3' 'MB:tma' 'COPY:' > gpurun_out/k1_c4.jsonl 2>gpurun_out/k1_c4.err; cat gpurun_out/k1_c4.jsonl
BATCH=1 SIZE=32768 ROUNDS=4 python tools/cmp_variants.py 8 'ANA:' 'ANA:FHWT_ANA_FUSED=8' 'ANA:FHWT_ANA_FUSED=8,FHWT_ANA_STAGES=3' > gpurun_out/k1_c5.jsonl 2>gpurun_out/k1_c5.err; cat gpurun_out/k1_c5.jsonl
