#!/bin/bash
# ncu --set full of kernels matching $2 in `python tools/prof_next.py`: summary, stall sampling, per-line attribution
TAG=$1; K=$2; N=${3:-4}
python tools/prof_next.py > /dev/null || exit 1
ncu -f --set full --clock-control none --import-source on -k regex:"$K" -c $N -o /tmp/k_$TAG python tools/prof_next.py > gpurun_out/ncu_k_$TAG.log 2>&1
python tools/ncu_summary.py /tmp/k_$TAG.ncu-rep > gpurun_out/k_$TAG.txt 2>&1
ncu -i /tmp/k_$TAG.ncu-rep --page raw --csv > /tmp/k_$TAG.csv 2>/dev/null
for r in $(seq 0 $((N - 1))); do python tools/ncu_stalls.py /tmp/k_$TAG.csv $r >> gpurun_out/k_$TAG.txt 2>&1; done
python tools/ncu_lines.py /tmp/k_$TAG.ncu-rep "${4:-$K}" 40 16588800 >> gpurun_out/k_$TAG.txt 2>&1
cat gpurun_out/k_$TAG.txt
