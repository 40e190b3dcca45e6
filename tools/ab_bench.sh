#!/bin/bash
# A/B of two library builds on the same box: alternating bench lines
# ALT=tools/ab/<lib>.so WL=c4a ROUNDS=2 bash tools/ab_bench.sh
for r in $(seq ${ROUNDS:-2}); do
  for v in new alt; do
    if [ $v = alt ]; then export SSB_LIB_PATH=$ALT; else unset SSB_LIB_PATH; fi
    for w in ${WL:-c4a}; do
      timeout 600 python bench.py --workload $w --steps ${STEPS:-10} --no-e2e --no-cpu --no-also 2>&1 | tail -1 | python -c "
import json,sys
l=sys.stdin.read()
try:
  d=json.loads(l); print('$v', d['config']['workload'][:12], d['value'], 'step_frac', d['step_roofline']['frac'], 'clk', d['clocks'].get('sm_mhz'), 'bwd_l0', d['kernels_ms'].get('bwd_l0'), 'bwd_l1', d['kernels_ms'].get('bwd_l1'), 'bwd_l2', d['kernels_ms'].get('bwd_l2'), 'fwd_l0', d['kernels_ms'].get('fwd_l0'), 'up', d['kernels_ms'].get('bwd_up'), 'pool', d['kernels_ms'].get('pool0->1'))
except Exception as e: print('ERR', l[-1500:])
"
    done
  done
done
