# Round-2 evidence refresh on the shipped kernels: GPU tests, smoke, default bench line, the launch
# list of the bench command, and full-size `ncu --set full` captures of K1/K4 (c4), K5 (c2), K1/K4 (c5)
# exported here as raw + source CSVs (tools/ncu_traffic.py, tools/sass_hotspots.py read them).
mkdir -p gpurun_out/ev
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/ev/pytest.log 2>&1; echo "pytest rc=$?" | tee -a gpurun_out/ev/pytest.log
tail -3 gpurun_out/ev/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/ev/bench.json 2> gpurun_out/ev/bench.err; echo "bench rc=$?"
tail -2 gpurun_out/ev/bench.err
B="python bench.py --steps 2 --warmup 3 --no-breakdown --no-direct --sustained 0"
$B > gpurun_out/ev/plain_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/ev/launches.csv $B > gpurun_out/ev/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
for spec in "c4 256 ana2d|syn2d" "c2 4096 ana1d|syn1d" "c5 32768 ana2d|syn2d"; do
  set -- $spec
  python tools/profile_case.py $1 $2 > gpurun_out/ev/plain_$1.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k "regex:$3" -c 2 -o gpurun_out/ev/full_$1 -f \
      python tools/profile_case.py $1 $2 > gpurun_out/ev/ncu_$1.log 2>&1; echo "ncu $1 rc=$?"
  ncu -i gpurun_out/ev/full_$1.ncu-rep --page raw --csv > gpurun_out/ev/raw_$1.csv 2>/dev/null
  ncu -i gpurun_out/ev/full_$1.ncu-rep --page source --csv --print-source sass > gpurun_out/ev/src_$1.csv 2>/dev/null
done
ls -la gpurun_out/ev
du -sh gpurun_out/ev
# keep the transfer under the 64 MiB cap: drop the c2/c5 reports (their CSVs are exported above)
rm -f gpurun_out/ev/full_c2.ncu-rep gpurun_out/ev/full_c5.ncu-rep
du -sh gpurun_out/ev
