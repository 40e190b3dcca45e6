#!/bin/bash
# ncu --set full of the 8(f) row kernels (second iteration of tools/prof_next.py), summarised on the box
set -x
TAG=${1:-next}
python -m paper_2602_08642_b200.build > gpurun_out/build_$TAG.log 2>&1 || exit 1
python tools/prof_next.py || exit 1
ncu --set full --clock-control none --import-source on \
    -f -k regex:"k_warp|k_motion|k_score|k_sg_|k_blur|k_sums|k_max_reduce|k_tonemap|k_loss|k_epilogue" -c 80 \
    -o /tmp/next_$TAG python tools/prof_next.py > gpurun_out/ncu_$TAG.log 2>&1
python tools/ncu_summary.py /tmp/next_$TAG.ncu-rep --stalls > gpurun_out/next_$TAG.txt 2>&1
cat gpurun_out/next_$TAG.txt
