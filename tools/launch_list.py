"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per-kernel count, total and mean device time, and share of the total.

    python tools/launch_list.py gpurun_out/launches.csv [--skip N]
"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    skip = int(sys.argv[sys.argv.index("--skip") + 1]) if "--skip" in sys.argv else 0
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    agg = collections.OrderedDict()
    n = 0
    for r in rows[1:]:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        n += 1
        if n <= skip:
            continue
        name = r[ix["Kernel Name"]]
        short = name.replace("void ", "").replace("ssb::", "").split("(")[0]
        unit = r[ix["Metric Unit"]]
        v = float(r[ix["Metric Value"]].replace(",", ""))
        us = v / 1e3 if unit == "ns" else (v * 1e3 if unit == "ms" else v)
        a = agg.setdefault(short, [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':72s} {'n':>4s} {'total us':>11s} {'mean us':>10s} {'share':>6s}")
    for k, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:72]:72s} {c:4d} {us:11.1f} {us / c:10.2f} {100 * us / tot:5.1f}%")
    print(f"{'TOTAL':72s} {sum(v[0] for v in agg.values()):4d} {tot:11.1f}")


if __name__ == "__main__":
    main()
