set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r2_smi.txt
free -g >> gpurun_out/r2_smi.txt; nproc >> gpurun_out/r2_smi.txt
timeout 2400 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider --durations=25 > gpurun_out/r2_pytest1.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest1.log
CFGS="4 2 2 256 60 120|4 3 2 256 44 120|4 3 2 256 36 120|4 3 2 256 28 120|4 4 2 256 28 120|4 3 1 256 60 120|4 3 2 256 44 240|4 3 1 512 60 120|8 2 1 512 60 120" 
IFS='|'; for c in $CFGS; do IFS=' '; CFGS="$c" timeout 120 bash tools/probe/pattern_sweep.sh; done > gpurun_out/r2_probe.txt 2>&1
