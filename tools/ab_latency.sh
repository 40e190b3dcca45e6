# same-box A/B of the latency lines (c1 / c0 / training placement): ALT=tools/ab/<lib>.so bash tools/ab_latency.sh
for r in 1 2; do
  for v in new alt; do
    if [ $v = alt ]; then export SSB_LIB_PATH=$ALT; else unset SSB_LIB_PATH; fi
    python tools/bench_latency.py | python -c "
import json,sys; d=json.load(sys.stdin)
print('$v', 'c1', d['c1']['us_per_frame'], 'place', d['c1']['placement_us'], 'c0', d['c0']['us_per_frame'], 'train', d['place_train']['mpix_s'])"
  done
done
