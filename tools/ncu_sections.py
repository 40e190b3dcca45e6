"""Group an ncu_lines.py listing by the `// ----` section markers of a source
file: per-section thread-instructions per pixel and stall share.

    python tools/ncu_sections.py LINES.txt SOURCE.cuh
"""
import re
import sys


def main():
    lines = open(sys.argv[1]).read().split("\n")[1:]
    src = open(sys.argv[2]).read().split("\n")
    base = sys.argv[2].split("/")[-1][:16]
    marks = [(i + 1, l.strip().strip("/- ")) for i, l in enumerate(src) if "// ----" in l or "// ====" in l]
    agg = {}
    for l in lines:
        m = re.match(r"(\S+)\s*:(\d+)\s+([\d.]+)%\s+([\d.]+)/px st\s+([\d.]+)%", l)
        if not m:
            continue
        f, ln, px, st = m.group(1), int(m.group(2)), float(m.group(4)), float(m.group(5))
        name = "helper:" + f
        if f.startswith(base[:12]):
            name = "(pre)"
            for mk, t in marks:
                if ln >= mk:
                    name = t
        a = agg.setdefault(name, [0.0, 0.0])
        a[0] += px
        a[1] += st
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"{k[:64]:64s} {v[0]:7.1f}/px  stall {v[1]:5.1f}%")


if __name__ == "__main__":
    main()
