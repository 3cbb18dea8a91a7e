export FHWT_TUNING=1
FHWT_ANA_FUSED=7 ncu --set full --clock-control none --import-source on -k regex:ana2d -c 1 -o gpurun_out/k1_fp7 -f python tools/profile_case.py c4 64 > gpurun_out/k1_ncu_fp7.log 2>&1; echo "rc=$?"
ncu -i gpurun_out/k1_fp7.ncu-rep --page raw --csv > gpurun_out/k1_fp7_raw.csv 2>/dev/null
ncu -i gpurun_out/k1_fp7.ncu-rep --page source --csv --print-source sass > gpurun_out/k1_fp7_sass.csv 2>/dev/null
ncu -i gpurun_out/k1_default.ncu-rep --page source --csv --print-source sass > gpurun_out/k1_default_sass.csv 2>/dev/null || true
rm -f gpurun_out/k1_fp7.ncu-rep
