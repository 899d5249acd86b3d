#!/usr/bin/env python
"""Key metrics of every kernel in an ncu report (raw page), for profiles/ notes.

    python tools/ncu_summary.py <report.ncu-rep> [units]

units (optional): work units of the profiled launch, to print warp
instructions per unit."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time_(ncu unit)", 1),
    ("smsp__inst_executed.sum", "warp_inst", 1),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct", 1),
    ("launch__registers_per_thread", "regs", 1),
    ("launch__occupancy_limit_registers", "occ_lim_regs", 1),
    ("launch__occupancy_limit_shared_mem", "occ_lim_smem", 1),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads_per_inst", 1),
    ("sm__inst_executed_pipe_fp64.sum.pct_of_peak_sustained_active", "fp64_pipe_pct", 1),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_pipe_pct", 1),
    ("sm__inst_executed_pipe_alu.sum.pct_of_peak_sustained_active", "alu_pipe_pct", 1),
    ("sm__inst_executed_pipe_xu.sum.pct_of_peak_sustained_active", "xu_pipe_pct", 1),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "l1_lsu_wavefronts_pct", 1),
    ("smsp__inst_executed_op_global_red.sum", "global_red", 1),
    ("lts__t_sectors_op_red.sum.pct_of_peak_sustained_elapsed", "l2_red_sectors_pct", 1),
    ("dram__bytes_read.sum", "dram_read_B", 1),
    ("dram__bytes_write.sum", "dram_write_B", 1),
]


def main():
    rep = sys.argv[1]
    units = float(sys.argv[2]) if len(sys.argv) > 2 else None
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    for v in rows[2:]:
        print(v[h.index("Kernel Name")][:90])
        stalls = {}
        for i, name in enumerate(h):
            if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("not_issued"):
                try:
                    stalls[name[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(v[i].replace(",", ""))
                except ValueError:
                    pass
        for key, label, scale in KEYS:
            if key in h:
                try:
                    x = float(v[h.index(key)].replace(",", "")) * scale
                except ValueError:
                    continue
                print(f"  {label:24s} {x:.4g}")
        if units and "smsp__inst_executed.sum" in h:
            wi = float(v[h.index("smsp__inst_executed.sum")].replace(",", ""))
            print(f"  {'warp_inst_per_unit':24s} {wi / units:.4g}")
        tot = sum(stalls.values()) or 1
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:8]
        print("  stalls: " + ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in top))


if __name__ == "__main__":
    main()
