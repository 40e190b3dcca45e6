"""bench.call_shapes alone (history / no-demod / C=12 call shapes)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

print(json.dumps(bench.call_shapes(6551.4)))
