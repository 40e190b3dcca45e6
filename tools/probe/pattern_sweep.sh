#!/bin/bash
# build + run the level-0 backward memory-pattern probe for a few stream shapes
cd "$(dirname "$0")"
for cfg in ${CFGS:-"4 2 2 256" "4 3 2 256" "4 4 1 256" "8 2 1 256" "8 2 1 512" "4 3 1 512" "4 2 1 256" "2 4 2 256"}; do
  set -- $cfg
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DPS=$1 -DNST=$2 -DMINB=$3 -DNTHR=$4 pattern_probe.cu \
       -o /tmp/pp_$1_$2_$3_$4 -lcuda 2>&1 | grep -i error
  /tmp/pp_$1_$2_$3_$4 16
done
