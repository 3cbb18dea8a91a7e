REPS=2 WL=c4 bash tools/bench_ab.sh "" "FHWT_LIB=paper_1002_2184_b200/libfhwt_nc.so" > gpurun_out/sweep17_c4.jsonl
cat gpurun_out/sweep17_c4.jsonl
FHWT_TUNING=1 FHWT_LIB=paper_1002_2184_b200/libfhwt_nc.so python bench.py --steps 5 --warmup 3 --no-breakdown --no-direct --sustained 0 --no-e2e --no-cpu-baseline 2>&1 | tail -2 | cut -c1-300
