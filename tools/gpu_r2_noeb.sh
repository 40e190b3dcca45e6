SSB_BWD_NOEB=1 timeout 900 python -m pytest tests/test_gpu_pyramid.py tests/test_gpu_fullsize.py -m gpu -q -x -k "tma or level0 or full_frame or golden or oracle or bf16" -p no:cacheprovider > gpurun_out/r2_noeb_tests.txt 2>&1
for r in 1 2; do for v in 0 1; do for w in c4a c3; do SSB_BWD_NOEB=$v python bench.py --workload $w --steps 10 --no-e2e --no-cpu --no-also 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('noeb=$v $w', d['value'], 'step_frac', d['step_roofline']['frac'], 'clk', d['clocks'].get('sm_mhz'), 'bwd_l0', d['kernels_ms'].get('bwd_l0'))"; done; done; done > gpurun_out/r2_noeb_bench.txt 2>&1
