# row-segment length sweep (SSB_SEG_ROWS) of the c4a / c3 bench lines
for sr in ${SEGS:-64 96 128}; do
  echo "SEG $sr"; SSB_SEG_ROWS=$sr WORKLOADS="${WL:-c4a c3}" bash tools/gpu_quick.sh 2>&1 | grep -E "^c4a|^c3" | cut -c1-120
done
