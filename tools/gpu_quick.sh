# quick GPU check: build, gpu tests, c4a + c3 bench lines (no e2e/cpu legs)
mkdir -p gpurun_out
python -m paper_2602_08642_b200.build > /dev/null || exit 1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for w in ${WORKLOADS:-c4a c3}; do
  timeout 600 python bench.py --workload $w --steps 10 --no-e2e --no-cpu --no-also 2>&1 | tail -1 | python -c "
import json,sys
l=sys.stdin.read()
try:
  d=json.loads(l); print(d['config']['workload'][:40], d['value'], d['unit'], 'step_frac', d['step_roofline']['frac'], 'bwd_l0_frac', d['roofline']['frac'], json.dumps(d['kernels_ms']))
except Exception as e: print('ERR', l[-2000:])
"
done
