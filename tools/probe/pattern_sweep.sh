#!/bin/bash
# build + run the level-0 backward memory-pattern probe for a few stream shapes
# CFGS: '|'-separated entries "S stages minb threads [txb [seg]]"
cd "$(dirname "$0")"
CFGS=${CFGS:-"4 2 2 256|4 3 2 256|4 4 1 256|8 2 1 256|8 2 1 512|4 3 1 512|4 2 1 256|2 4 2 256"}
IFS='|' read -ra LIST <<< "$CFGS"
for cfg in "${LIST[@]}"; do
  set -- $cfg
  txb=${5:-60}; seg=${6:-120}
  bin=/tmp/pp_$1_$2_$3_$4_${txb}_$seg
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DPS=$1 -DNST=$2 -DMINB=$3 -DNTHR=$4 -DPTXB=$txb -DPSEG=$seg \
       pattern_probe.cu -o $bin -lcuda 2>&1 | grep -i error
  timeout 60 $bin ${FRAMES:-16}
done
