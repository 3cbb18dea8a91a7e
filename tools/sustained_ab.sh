#!/bin/bash
# Interleaved A/B of library builds / knobs on the c4 step, burst (graph replays, 20 steps) and
# power-capped (the bench's `sustained` block: 1.5 s back to back, then 1.5 s timed):
#   REPS=3 bash tools/sustained_ab.sh "" "FHWT_LIB=$PWD/paper_1002_2184_b200/libX.so" ...
export FHWT_TUNING=1
B="python bench.py --workload c4 --steps 20 --warmup 5 --no-breakdown --no-direct --no-e2e --no-cpu-baseline --no-t1 --sustained 1.5"
for i in $(seq 1 ${REPS:-3}); do
  for cfg in "$@"; do
    env $cfg $B 2>/dev/null | tail -1 | CFG="$cfg" python -c "
import json, os, sys
d = json.loads(sys.stdin.read()); k = d['kernels']; s = d['sustained']['default']
print(json.dumps({'cfg': os.environ['CFG'].split('/')[-1], 'value': round(d['value']), 'ana': round(k['analysis_gbs']),
                  'syn': round(k['synthesis_gbs']), 'sustained': round(s['value']), 'sus_mhz': s.get('sm_mhz_median'),
                  'sus_w': s.get('power_w_median')}))"
  done
done
