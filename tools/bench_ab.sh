#!/bin/bash
# Interleaved A/B of library knobs in the bench's own timing context (CUDA-graph DWT+IDWT steps):
#   REPS=3 WL=c4 bash tools/bench_ab.sh "" "FHWT_ANA_L2HINT=0" "FHWT_SYN_L2MODE=1 FHWT_ANA_L2HINT=0" ...
# one JSON line per run: the knob set, DWT+IDWT GB/s, analysis / synthesis GB/s (CUDA events), SM clock.
export FHWT_TUNING=1
WL=${WL:-c4}
B="python bench.py --workload $WL --steps 20 --warmup 5 --no-breakdown --no-direct --sustained 0 --no-e2e --no-cpu-baseline --no-t1"
for i in $(seq 1 ${REPS:-3}); do
  for cfg in "$@"; do
    env $cfg $B 2>/dev/null | tail -1 | CFG="$cfg" python -c "
import json, os, sys
d = json.loads(sys.stdin.read()); k = d['kernels']
print(json.dumps({'wl': '$WL', 'cfg': os.environ['CFG'], 'value': round(d['value']), 'ana': round(k['analysis_gbs']),
                  'syn': round(k['synthesis_gbs']), 'clk': d['clocks'].get('sm_mhz'), 'reasons': d['clocks'].get('reasons')}))"
  done
done
