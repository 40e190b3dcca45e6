"""Top SASS instructions by stall samples (with the dominant reasons) from an
`ncu --page source --csv --print-source sass` dump.

    python tools/sass_stalls.py DUMP.csv [TOP]
"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    hdr = rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    body = [r for r in rows[2:] if len(r) == len(hdr)]
    tot = sum(int(r[idx["Warp Stall Sampling (All Samples)"]] or 0) for r in body)
    body.sort(key=lambda r: -int(r[idx["Warp Stall Sampling (All Samples)"]] or 0))
    print(f"total samples {tot}")
    for k, r in enumerate(body[:top]):
        s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        reasons = sorted(((int(r[idx[c]] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
        rs = " ".join(f"{n}:{v * 100 / max(s, 1):.0f}%" for v, n in reasons if v)
        pos = next(i for i, rr in enumerate(rows[2:]) if rr is r) if False else ""
        print(f"{s * 100 / tot:5.2f}%  {r[idx['Address']][-5:]}  {r[idx['Source']].strip()[:60]:60s} {rs}")


if __name__ == "__main__":
    main()
