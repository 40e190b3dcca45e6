# SSB_MIN_CTAS_SMALL sweep on the small-level-heavy workloads (c3, c2)
for v in 0 296 592 0 296 592; do
  for w in c3 c2; do
    SSB_MIN_CTAS_SMALL=$v timeout 600 python bench.py --workload $w --steps 10 --no-e2e --no-cpu --no-also 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels_ms']
print('$v', '$w', d['value'], d['step_roofline']['frac'], {n: k.get(n) for n in ('bwd_l1','bwd_l2','bwd_l3','fwd_l2','fwd_l3','fwd_l1')})"
  done
done
