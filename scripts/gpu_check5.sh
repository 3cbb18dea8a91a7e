python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/c5_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c5_pytest.log; tail -2 gpurun_out/c5_pytest.log
timeout 900 python tools/stress_parity.py 800 31337 > gpurun_out/c5_stress.log 2>&1; echo "stress rc=$?"; tail -2 gpurun_out/c5_stress.log
REPS=2 WL=c4 bash tools/bench_ab.sh "" > gpurun_out/c5_ab.jsonl; cat gpurun_out/c5_ab.jsonl
