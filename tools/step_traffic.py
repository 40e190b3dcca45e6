"""Per-kernel DRAM traffic of one pyramid fwd+bwd step from an ncu metrics
list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--csv), restricted to this repo's kernels and the LAST step of the capture.

    python tools/step_traffic.py LAUNCHES.csv PIXELS_PER_STEP [PEAK_GBS]

Prints each launch (duration, DRAM bytes, GB/s) and the step totals: DRAM
bytes per pixel and the time-weighted achieved bandwidth (sum bytes / sum
durations -- serialized, cold-cache ncu launches, so a lower bound on the
live rate)."""
import collections
import csv
import json
import re
import sys

OURS = re.compile(r"k_pyr_|k_up_transpose|k_pool_chain|k_pool2")


def main():
    path, px = sys.argv[1], float(sys.argv[2])
    peak = float(sys.argv[3]) if len(sys.argv) > 3 else 6551.4
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    launches = collections.OrderedDict()
    for r in rows[1:]:
        name = r[ix["Kernel Name"]]
        if not OURS.search(name):
            continue
        d = launches.setdefault(r[ix["ID"]], {"name": name})
        unit, v = r[ix["Metric Unit"]], float(r[ix["Metric Value"]].replace(",", ""))
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3,
                 "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)
        d[r[ix["Metric Name"]]] = v * scale
    ls = list(launches.values())
    # the last step: from the last pool launch before the last forward sweep
    starts = [i for i, d in enumerate(ls) if "k_pool2" in d["name"]]
    first = starts[0] if starts else 0
    for i in range(1, len(starts)):
        if starts[i] != starts[i - 1] + 1:
            first = starts[i]
    step = ls[first:]
    tot_us = tot_b = 0.0
    print(f"{'kernel':64s} {'us':>9s} {'MB':>9s} {'GB/s':>7s} {'B/px':>7s}")
    out = []
    for d in step:
        us = d.get("gpu__time_duration.sum", 0.0)
        b = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        tot_us += us
        tot_b += b
        short = d["name"].replace("void ", "").replace("ssb::", "").split("(")[0]
        print(f"{short[:64]:64s} {us:9.1f} {b / 1e6:9.1f} {b / (us * 1e-6) / 1e9 if us else 0:7.0f} {b / px:7.1f}")
        out.append({"kernel": short, "us": round(us, 2), "bytes": int(b)})
    gbs = tot_b / (tot_us * 1e-6) / 1e9
    print(f"{'STEP':64s} {tot_us:9.1f} {tot_b / 1e6:9.1f} {gbs:7.0f} {tot_b / px:7.1f}   "
          f"({100 * gbs / peak:.1f}% of {peak:.0f} GB/s)")
    print(json.dumps({"dram_bytes_per_px": round(tot_b / px, 2), "launches": len(step)}))


if __name__ == "__main__":
    main()
