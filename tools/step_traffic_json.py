"""profiles/step_traffic.json (read by bench.py `step_dram`) from the output
of tools/gpu_step_traffic.sh.

    python tools/step_traffic_json.py gpurun_out/TAG_step_traffic.txt > profiles/step_traffic.json
"""
import json
import sys

parts = open(sys.argv[1]).read().split("\n\n")
tag = sys.argv[1].split("/")[-1]
out = {}
for part, wl, src in ((parts[0], "c4a", "4 x 1920x1080 L3 k5 fp32"), (parts[1], "c3", "1 x 3840x2160 L4 k7 bf16")):
    j = json.loads(part.strip().split("\n")[-1])
    out[wl] = {"dram_bytes_per_px": j["dram_bytes_per_px"], "launches": j["launches"],
               "source": f"ncu --metrics dram__bytes_read/write.sum of every kernel of one {src} step "
                         f"(tools/gpu_step_traffic.sh, profiles/{tag})"}
print(json.dumps(out, indent=1))
