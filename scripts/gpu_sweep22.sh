for wl in c4 c5; do
REPS=3 WL=$wl bash tools/bench_ab.sh "" "FHWT_LIB=paper_1002_2184_b200/libfhwt_prodB.so" > gpurun_out/sweep22_$wl.jsonl
cat gpurun_out/sweep22_$wl.jsonl
done
