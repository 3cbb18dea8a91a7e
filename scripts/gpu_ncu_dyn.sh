mkdir -p gpurun_out/ncu2
python tools/profile_case.py c4 256 > gpurun_out/ncu2/plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:ana2d|syn2d" -c 2 -o gpurun_out/ncu2/full_c4 -f \
    python tools/profile_case.py c4 256 > gpurun_out/ncu2/ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
ncu -i gpurun_out/ncu2/full_c4.ncu-rep --page raw --csv > gpurun_out/ncu2/raw_c4.csv 2>/dev/null
for k in ana2d syn2d; do ncu -i gpurun_out/ncu2/full_c4.ncu-rep --page source --csv --print-source sass -k regex:$k > gpurun_out/ncu2/src_c4_$k.csv 2>/dev/null; done
python tools/profile_case.py c5 32768 > gpurun_out/ncu2/plain_c5.log 2>&1 && \
ncu --set full --clock-control none -k "regex:ana2d|syn2d" -c 2 -o gpurun_out/ncu2/full_c5 -f \
    python tools/profile_case.py c5 32768 > gpurun_out/ncu2/ncu_c5.log 2>&1; echo "ncu c5 rc=$?"
ncu -i gpurun_out/ncu2/full_c5.ncu-rep --page raw --csv > gpurun_out/ncu2/raw_c5.csv 2>/dev/null
rm -f gpurun_out/ncu2/full_c5.ncu-rep
ls -la gpurun_out/ncu2
