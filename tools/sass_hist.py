"""Opcode histogram (executed warp instructions, stall samples) of an ncu
`--page source --csv --print-source sass` export.

    python tools/sass_hist.py EXPORT.csv [PIXELS] [TOP]
"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    px = float(sys.argv[2]) if len(sys.argv) > 2 else 0
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    ex, st = collections.Counter(), collections.Counter()
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        op = r[ix["Source"]].strip().split()
        if not op:
            continue
        o = op[0]
        if o.startswith("@"):
            o = op[1]
        o = o.split(".")[0] + ("." + o.split(".")[1] if o.startswith(("LDS", "STS", "LDG", "STG")) and "." in o else "")
        ex[o] += float(r[ix["Instructions Executed"]] or 0)
        st[o] += float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    tot, stot = sum(ex.values()), sum(st.values())
    print(f"total warp instr {tot:.4g}" + (f"  per px {tot / px:.2f}" if px else ""))
    for o, v in ex.most_common(top):
        print(f"{o:12s} {v:12.4g} {100 * v / tot:5.1f}%" + (f" {v / px:7.2f}/px" if px else "") +
              f"   stalls {100 * st[o] / stot:5.1f}%")


if __name__ == "__main__":
    main()
