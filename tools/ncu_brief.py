"""One-line-per-kernel summary of an ncu --set full report (duration, pipes, issue,
occupancy, shared-memory wavefronts, top stall reasons): tools/ncu_brief.py REP"""
import csv
import subprocess
import sys

W = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
     "smsp__issue_active.avg.pct_of_peak_sustained_active",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
     "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
     "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    stall = [(i, x) for i, x in enumerate(h)
             if x.startswith("smsp__pcsamp_warps_issue_stalled") and not x.endswith("not_issued")]
    for r in rows[2:]:
        print(r[h.index("Kernel Name")].split("(")[0], r[h.index("Grid Size")])
        for w in W:
            if w in h:
                i = h.index(w)
                print(f"  {w} = {r[i]} {units[i]}")
        top = sorted(((float(r[i].replace(",", "") or 0), x[33:]) for i, x in stall), reverse=True)[:6]
        print("  stalls:", ", ".join(f"{n} {v:.0f}" for v, n in top))


if __name__ == "__main__":
    main(sys.argv[1])
