REPS=2 WL=c4 bash tools/bench_ab.sh "" "FHWT_LIB=paper_1002_2184_b200/libfhwt_ncmp.so" "FHWT_LIB=paper_1002_2184_b200/libfhwt_ncmp.so FHWT_SYN_STAGES=2" "FHWT_LIB=paper_1002_2184_b200/libfhwt_ncmp.so FHWT_SYN_PROD=0" > gpurun_out/sweep18_c4.jsonl
cat gpurun_out/sweep18_c4.jsonl
