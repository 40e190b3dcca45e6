"""Shared-memory wavefronts and bank-conflict replays per CUDA source line of
one kernel: an `ncu --page source --csv --print-source sass` dump mapped to
lines through `nvdisasm -g` of the kernel's cubin (same build).

    python tools/smem_lines.py DUMP.csv OBJ.o MANGLED_NAME [TOP]
"""
import csv
import os
import re
import subprocess
import sys
import tempfile


def main():
    dump, obj, fn = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 20
    with tempfile.TemporaryDirectory() as td:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=td, capture_output=True)
        head = f".text.{fn}:"
        for cub in sorted(f for f in os.listdir(td) if f.endswith(".cubin")):
            if fn.encode() not in open(os.path.join(td, cub), "rb").read():
                continue
            lines = subprocess.run(["nvdisasm", "-g", os.path.join(td, cub)], capture_output=True,
                                   text=True).stdout.splitlines()
            hits = [i for i, l in enumerate(lines) if l.strip() == head]
            if hits:
                start = hits[0]
                break
    cur, off2line = None, {}
    for l in lines[start + 1:]:
        s = l.strip()
        if s.startswith(".text.") and s.endswith(":"):
            break
        m = re.search(r'## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
        if m and cur:
            off2line[int(m.group(1), 16)] = cur
    rows = list(csv.reader(open(dump)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    body = [r for r in rows[2:] if len(r) == len(hdr)]
    base = int(body[0][ix["Address"]], 16)
    f = lambda r, k: float(r[ix[k]] or 0)  # noqa: E731
    agg, tot, exc = {}, 0.0, 0.0
    for r in body:
        w, e = f(r, "L1 Wavefronts Shared"), f(r, "L1 Wavefronts Shared Excessive")
        a = agg.setdefault(off2line.get(int(r[ix["Address"]], 16) - base, ("?", 0)), [0.0, 0.0])
        a[0] += w
        a[1] += e
        tot += w
        exc += e
    print(f"shared wavefronts {tot:.3e}, bank-conflict replays {exc:.3e} ({100 * exc / max(tot, 1):.1f}%)")
    srcs = {}
    for (fname, ln), (w, e) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        if fname not in srcs:
            p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2602_08642_b200", "csrc", fname)
            srcs[fname] = open(p).read().splitlines() if os.path.exists(p) else []
        txt = srcs[fname][ln - 1].strip()[:64] if 0 < ln <= len(srcs[fname]) else ""
        print(f"{fname}:{ln:<5d} wavefronts {100 * w / tot:5.2f}%  replays {100 * e / tot:5.2f}%  {txt}")


if __name__ == "__main__":
    main()
