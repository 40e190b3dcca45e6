"""Warp-stall sampling breakdown (+ a few key metrics) from an ncu raw csv.

    python tools/ncu_stalls.py RAW.csv [ROW]
"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    hdr, units, r = rows[0], rows[1], rows[2 + k]
    print(r[hdr.index("Kernel Name")][:90])
    st = []
    for i, h in enumerate(hdr):
        if "pcsamp_warps_issue_stalled" in h and "not_issued" not in h:
            try:
                st.append((float(r[i].replace(",", "")), h))
            except ValueError:
                pass
    st.sort(reverse=True)
    tot = sum(v for v, _ in st) or 1
    for v, h in st[:10]:
        print(f"  {h.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {100 * v / tot:5.1f}%")
    for key in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
                "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
                "smsp__issue_active.avg.pct_of_peak_sustained_active"]:
        if key in hdr:
            print(f"  {key:55s} {r[hdr.index(key)]} {units[hdr.index(key)]}")


if __name__ == "__main__":
    main()
