#!/bin/bash
# A/B of the level-0 backward variants (SSB_BWD0=<stages>,<own columns>):
# parity subset first, then the bench line per variant.
# VARS="0 3,32 ..." WL="c4a" bash tools/variant_sweep.sh
mkdir -p gpurun_out
for v in ${VARS:-0}; do
  echo "== SSB_BWD0=$v"
  SSB_BWD0=$v timeout 600 python -m pytest tests/test_gpu_pyramid.py tests/test_gpu_fullsize.py -m gpu -q -x \
     -k "${TESTK:-tma or level0 or bf16 or full_frame}" -p no:cacheprovider 2>&1 | tail -2
  for w in ${WL:-c4a}; do
    SSB_BWD0=$v timeout 600 python bench.py --workload $w --steps ${STEPS:-10} --no-e2e --no-cpu --no-also 2>&1 | tail -1 | python -c "
import json,sys
l=sys.stdin.read()
try:
  d=json.loads(l); print('$v', d['config']['workload'][:12], d['value'], d['unit'], 'step_frac', d['step_roofline']['frac'], 'bwd_l0_frac', d['roofline']['frac'], 'clk', d['clocks'].get('sm_mhz'), json.dumps(d['kernels_ms']))
except Exception as e: print('ERR', l[-2000:])
"
  done
done
