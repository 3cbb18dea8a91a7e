#!/bin/bash
# Full-size ncu captures of the c4 / c5 bench kernels (K1 ana2d_lean, K4 syn2d_prod), exported on the
# box to CSV (raw counters + SASS source page) so gpurun_out/ stays small:
#   bash tools/ncu_k4k1.sh <tag>   -> gpurun_out/<tag>_<wl>_<kernel>_{raw,src}.csv
T=${1:-ncu}
mkdir -p gpurun_out
for wl in "c4 256" "c5 32768"; do
  set -- $wl
  for k in syn2d_prod ana2d_lean; do
    rep=/tmp/${T}_$1_$k
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -f -o $rep \
      python tools/profile_case.py $1 $2 > gpurun_out/${T}_$1_${k}.log 2>&1
    ncu -i $rep.ncu-rep --page raw --csv > gpurun_out/${T}_$1_${k}_raw.csv 2>/dev/null
    ncu -i $rep.ncu-rep --page source --csv --print-source sass > gpurun_out/${T}_$1_${k}_src.csv 2>/dev/null
    ncu -i $rep.ncu-rep --page details --csv > gpurun_out/${T}_$1_${k}_details.csv 2>/dev/null
    rm -f $rep.ncu-rep
  done
done
ls -la gpurun_out
