"""Summarise an ncu --set full report: per kernel duration, DRAM bytes, L2 bytes, issue activity and
the top warp-stall reasons (used to write profiles/*.md and bench.py's `traffic`)."""
import csv
import subprocess
import sys


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return r[0], r[2:]


def main(rep):
    hdr, data = rows(rep)
    col = {h: i for i, h in enumerate(hdr)}

    def g(r, k):
        try:
            return float(r[col[k]].replace(",", ""))
        except (KeyError, ValueError):
            return float("nan")
    for r in data:
        name = r[col["Kernel Name"]].split("(")[0]
        dur = g(r, "gpu__time_duration.sum")
        dram = g(r, "dram__bytes_read.sum") + g(r, "dram__bytes_write.sum")
        print(f"== {name}  grid={r[col['launch__grid_size']]} block={r[col['launch__block_size']]} "
              f"regs={r[col['launch__registers_per_thread']]} dur={dur:.3f} (unit as reported)")
        for k in ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "smsp__inst_executed.sum",
                  "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
                  "lts__t_sectors_srcunit_tex_op_read.sum", "l1tex__t_bytes.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
                  "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
                  "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active" ]:
            if k in col:
                print(f"   {k:70s} {r[col[k]]}")
        st = [(h, g(r, h)) for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
        tot = sum(v for _, v in st if v == v)
        st.sort(key=lambda x: -x[1] if x[1] == x[1] else 0)
        print("   stalls: " + ", ".join(f"{h.replace('smsp__pcsamp_warps_issue_stalled_', '')}={100 * v / tot:.0f}%"
                                         for h, v in st[:7]))


if __name__ == "__main__":
    main(sys.argv[1])
