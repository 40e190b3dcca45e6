# minimum-CTA-count sweep (SSB_MIN_CTAS) of the c3 / c4a / c2 bench lines
for m in ${MINS:-1184 592 296}; do
  echo "MIN_CTAS $m"; SSB_MIN_CTAS=$m WORKLOADS="${WL:-c3 c4a}" bash tools/gpu_quick.sh 2>&1 | grep -E "^c4a|^c3|^c2" | cut -c1-400
done
