mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_pyramid.py tests/test_gpu_reference_suite.py -m gpu -q -rfE -p no:cacheprovider -s > gpurun_out/r2_pytest2.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest2.log
CFGS="4 2 2 256 60 120|4 3 2 256 44 120|4 3 2 256 36 120|4 3 2 256 28 120|4 4 2 256 28 120|4 3 1 256 60 120|4 3 2 256 44 240|4 3 1 512 60 120|8 2 1 512 60 120|4 3 2 256 40 120|4 3 2 256 32 120" bash tools/probe/pattern_sweep.sh > gpurun_out/r2_probe.txt 2>&1
