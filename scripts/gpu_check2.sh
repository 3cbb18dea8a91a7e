nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/c2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c2_pytest.log; tail -3 gpurun_out/c2_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c2_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/c2_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/c2_bench.json 2> gpurun_out/c2_bench.err; echo "bench rc=$?"
tail -2 gpurun_out/c2_bench.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/c2_bench.json').read().strip().splitlines()[-1])
print({k: d.get(k) for k in ('value','ms_per_step','gpu_launches')}, d['roofline'], d['clocks'], d['kernels'])
for w,b in d.get('workloads',{}).items(): print(w, round(b['value']), round(b['analysis_gbs']), round(b['synthesis_gbs']))
print(d.get('parity'))
PY
