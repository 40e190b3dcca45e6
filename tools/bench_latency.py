"""c1 / c0 latency + placement lines alone (bench.latency_configs)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

peak = json.load(open("MEASURED_PEAKS.json")).get("hbm_gbs", 6551.4) if os.path.exists("MEASURED_PEAKS.json") else 6551.4
print(json.dumps(bench.latency_configs(peak)))
