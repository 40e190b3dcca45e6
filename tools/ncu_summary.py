"""Summarise an ncu report: per-kernel duration, DRAM bytes/throughput, IPC,
occupancy and the top warp-stall reasons.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--stalls]
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "launch__grid_size"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return hdr, units, rows[2:]


def main():
    rep = sys.argv[1]
    hdr, units, rows = raw(rep)
    col = {h: i for i, h in enumerate(hdr)}
    for r in rows:
        name = r[col["Kernel Name"]]
        short = name.split("(")[0].replace("void ssb::", "")
        args = name[name.find("<"):name.find(">") + 1] if "<" in name else ""
        v = {k: r[col[k]] if k in col else "?" for k in KEYS}

        def f(k, scale=1.0):
            try:
                return float(v[k].replace(",", "")) * scale
            except ValueError:
                return float("nan")
        dur_us = f("gpu__time_duration.sum") / 1e3 if units[col["gpu__time_duration.sum"]] == "ns" else f("gpu__time_duration.sum")
        rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
        ru, wu = units[col["dram__bytes_read.sum"]], units[col["dram__bytes_write.sum"]]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd *= scale.get(ru, 1)
        wr *= scale.get(wu, 1)
        print(f"{short[:12]:12s} {args[:44]:44s} {dur_us:9.1f}us  dram {(rd + wr) / 1e6:8.1f}MB "
              f"{(rd + wr) / (dur_us * 1e-6) / 1e9:7.0f}GB/s ({f('dram__throughput.avg.pct_of_peak_sustained_elapsed'):5.1f}%) "
              f"issue {f('smsp__issue_active.avg.pct_of_peak_sustained_active'):5.1f}% "
              f"occ {f('sm__warps_active.avg.pct_of_peak_sustained_active'):5.1f}% regs {v['launch__registers_per_thread']}")
        if "--stalls" in sys.argv:
            stalls = [(h.replace("smsp__average_warp_latency_issue_stalled_", "").replace(".ratio", ""),
                       r[i]) for h, i in col.items()
                      if h.startswith("smsp__average_warp_latency_issue_stalled_") and h.endswith(".ratio")]
            vals = []
            for nm, x in stalls:
                try:
                    vals.append((float(x), nm))
                except ValueError:
                    pass
            vals.sort(reverse=True)
            print("    stalls (cycles/instr):", ", ".join(f"{nm}={x:.2f}" for x, nm in vals[:7]))


if __name__ == "__main__":
    main()
