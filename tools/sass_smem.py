"""Shared-memory wavefronts per SASS instruction (total, ideal, excessive =
bank-conflict replays) from an `ncu --page source --csv --print-source sass`
dump, with the CUDA source line when the dump carries it.

    python tools/sass_smem.py DUMP.csv [TOP]
"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    body = [r for r in rows[2:] if len(r) == len(hdr)]
    f = lambda r, k: float(r[ix[k]] or 0)  # noqa: E731
    tot = sum(f(r, "L1 Wavefronts Shared") for r in body)
    exc = sum(f(r, "L1 Wavefronts Shared Excessive") for r in body)
    print(f"shared wavefronts {tot:.3e}, excessive (bank conflicts) {exc:.3e} ({100 * exc / max(tot, 1):.1f}%)")
    body.sort(key=lambda r: -f(r, "L1 Wavefronts Shared"))
    for r in body[:top]:
        w, e, i = f(r, "L1 Wavefronts Shared"), f(r, "L1 Wavefronts Shared Excessive"), f(r, "L1 Wavefronts Shared Ideal")
        print(f"{100 * w / tot:5.2f}%  exc {100 * e / max(w, 1):5.1f}%  {r[ix['Address']][-5:]}  {r[ix['Source']].strip()[:70]}")


if __name__ == "__main__":
    main()
