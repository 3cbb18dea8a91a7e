python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/c3_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c3_pytest.log; tail -3 gpurun_out/c3_pytest.log
timeout 900 python tools/stress_parity.py 600 2026 > gpurun_out/c3_stress.log 2>&1; echo "stress rc=$?"; tail -4 gpurun_out/c3_stress.log
