# ncu evidence for the shipped kernels (launch list of the bench command; full-size --set full of
# K1/K4 (c4, c5) and K5 (c2)); raw + per-kernel source CSVs exported on the box
mkdir -p gpurun_out/ev2
B="python bench.py --steps 2 --warmup 3 --no-breakdown --no-direct --sustained 0"
$B > gpurun_out/ev2/plain_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/ev2/launches.csv $B > gpurun_out/ev2/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
for spec in "c4 256 ana2d|syn2d" "c2 4096 ana1d|syn1d" "c5 32768 ana2d|syn2d"; do
  set -- $spec
  python tools/profile_case.py $1 $2 > gpurun_out/ev2/plain_$1.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k "regex:$3" -c 2 -o gpurun_out/ev2/full_$1 -f \
      python tools/profile_case.py $1 $2 > gpurun_out/ev2/ncu_$1.log 2>&1; echo "ncu $1 rc=$?"
  ncu -i gpurun_out/ev2/full_$1.ncu-rep --page raw --csv > gpurun_out/ev2/raw_$1.csv 2>/dev/null
  for k in ana syn; do
    ncu -i gpurun_out/ev2/full_$1.ncu-rep --page source --csv --print-source sass -k regex:$k > gpurun_out/ev2/src_$1_$k.csv 2>/dev/null
  done
  rm -f gpurun_out/ev2/full_$1.ncu-rep
done
ls -la gpurun_out/ev2; du -sh gpurun_out/ev2
