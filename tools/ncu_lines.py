"""Per-source-line instruction / stall attribution for one kernel of an ncu
report (needs -lineinfo builds and --import-source on).

    python tools/ncu_lines.py REPORT KERNEL_REGEX [TOP] [PIXELS] [--by-stall]
"""
import collections
import csv
import io
import re
import subprocess
import sys


def main():
    rep, pat = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    pixels = float(sys.argv[4]) if len(sys.argv) > 4 else 0
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    per = collections.defaultdict(lambda: [0, 0, ""])
    fname, hdr, func, seen = None, None, "", []
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] in ("Function Name", "Kernel Name"):
            func = r[1]
            continue
        if not re.search(pat, func):
            continue
        if func not in seen:
            seen.append(func)
        if func != seen[0]:
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if not hdr or len(r) < 8 or not r[0].isdigit():
            continue
        ie = hdr.index("Instructions Executed")
        st = hdr.index("Warp Stall Sampling (All Samples)")
        try:
            n, s = int(r[ie] or 0), int(r[st] or 0)
        except ValueError:
            continue
        k = (fname, int(r[0]))
        per[k][0] += n
        per[k][1] += s
        per[k][2] = r[1]
    tot = sum(v[0] for v in per.values()) or 1
    tots = sum(v[1] for v in per.values()) or 1
    print(f"total warp-instructions {tot}" + (f"  ({tot * 32 / pixels:.0f} thread-instr/px)" if pixels else ""))
    key = (lambda kv: -kv[1][1]) if "--by-stall" in sys.argv else (lambda kv: -kv[1][0])
    for k, v in sorted(per.items(), key=key)[:top]:
        extra = f" {v[0] * 32 / pixels:6.1f}/px" if pixels else ""
        print(f"{k[0][:16]:16s}:{k[1]:<5d} {100 * v[0] / tot:5.1f}%{extra} st {100 * v[1] / tots:5.1f}%  {v[2].strip()[:80]}")


if __name__ == "__main__":
    main()
