REPS=2 WL=c4 bash tools/bench_ab.sh "" > gpurun_out/c4_ab.jsonl; cat gpurun_out/c4_ab.jsonl
REPS=1 WL=c5 bash tools/bench_ab.sh "" >> gpurun_out/c4_ab.jsonl; tail -1 gpurun_out/c4_ab.jsonl
timeout 1200 python tools/stress_parity.py 2500 99 > gpurun_out/c4_stress.log 2>&1; echo "stress rc=$?"; tail -3 gpurun_out/c4_stress.log
