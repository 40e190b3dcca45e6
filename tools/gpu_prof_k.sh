#!/bin/bash
# ncu --set full of kernels matching $2 (count $3, line filter $4): summary, stall sampling, per-line attribution.
# Workload: $CASE (default `tools/prof_next.py`; e.g. CASE="tools/prof_case.py --frames 4 --iters 2"), skip $SKIP launches.
TAG=$1; K=$2; N=${3:-4}
CASE=${CASE:-tools/prof_next.py}
PX=${PX:-16588800}
python $CASE > /dev/null || exit 1
ncu -f --set full --clock-control none --import-source on -k regex:"$K" -s ${SKIP:-0} -c $N -o /tmp/k_$TAG python $CASE > gpurun_out/ncu_k_$TAG.log 2>&1
python tools/ncu_summary.py /tmp/k_$TAG.ncu-rep > gpurun_out/k_$TAG.txt 2>&1
ncu -i /tmp/k_$TAG.ncu-rep --page raw --csv > /tmp/k_$TAG.csv 2>/dev/null
for r in $(seq 0 $((N - 1))); do python tools/ncu_stalls.py /tmp/k_$TAG.csv $r >> gpurun_out/k_$TAG.txt 2>&1; done
python tools/ncu_lines.py /tmp/k_$TAG.ncu-rep "${4:-$K}" 40 $PX >> gpurun_out/k_$TAG.txt 2>&1
cat gpurun_out/k_$TAG.txt
