P=paper_1002_2184_b200
for wl in c4 c5; do
REPS=2 WL=$wl bash tools/bench_ab.sh "" "FHWT_LIB=$P/libfhwt_pm3.so" "FHWT_LIB=$P/libfhwt_nu.so" "FHWT_LIB=$P/libfhwt_pm3nu.so" > gpurun_out/sweep24_$wl.jsonl
cat gpurun_out/sweep24_$wl.jsonl
done
