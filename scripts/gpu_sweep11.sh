P=paper_1002_2184_b200
for wl in c4 c2; do
REPS=2 WL=$wl bash tools/bench_ab.sh "" "FHWT_LIB=$P/libfhwt_stg1.so" "FHWT_LIB=$P/libfhwt_stg2.so" "FHWT_LIB=$P/libfhwt_stg3.so" "FHWT_LIB=$P/libfhwt_stg4.so" > gpurun_out/sweep11_$wl.jsonl
cat gpurun_out/sweep11_$wl.jsonl
done
