"""Per-kernel DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) from an
ncu `--page raw --csv` export, per frame of the captured workload, merged into
profiles/ncu_traffic.json (read by bench.py for `roofline.traffic`).

    python tools/ncu_traffic.py RAW.csv WORKLOAD FRAMES NAME=REGEX [NAME=REGEX ...] [--source TEXT]
"""
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main():
    args = [a for a in sys.argv[1:]]
    src = None
    if "--source" in args:
        i = args.index("--source")
        src = args[i + 1]
        del args[i:i + 2]
    path, workload, frames = args[0], args[1], int(args[2])
    pats = dict(a.split("=", 1) for a in args[3:])
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    out_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    db = json.load(open(out_path)) if os.path.exists(out_path) else {}
    entry = db.setdefault(workload, {})
    for name, pat in pats.items():
        for r in rows[2:]:
            if re.search(pat, r[ix["Kernel Name"]]):
                b = 0.0
                for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                    b += float(r[ix[m]].replace(",", "")) * SCALE.get(units[ix[m]], 1)
                entry[name] = {"bytes_per_frame": round(b / frames), "kernel": r[ix["Kernel Name"]][:80],
                               "source": src or os.path.basename(path)}
                break
    json.dump(db, open(out_path, "w"), indent=1, sort_keys=True)
    print(json.dumps(entry, indent=1))


if __name__ == "__main__":
    main()
