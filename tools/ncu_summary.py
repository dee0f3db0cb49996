#!/usr/bin/env python
"""Summarise an ncu report (read here, no GPU): per kernel launch the key
throughput, occupancy, pipe and stall metrics.  Usage: ncu_summary.py REP"""
import csv
import io
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "dur_us",   # printed as dur_ms (base unit ns)
    "launch__grid_size": "grid",
    "launch__registers_per_thread": "regs",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occ%",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram%",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64%",
    "sm__inst_executed.avg.per_cycle_active": "ipc",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue%",
    "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum": "local_ld_sect",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum": "dfma",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum": "dmul",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum": "dadd",
}
STALLS = ["no_instructions", "long_scoreboard", "short_scoreboard", "wait", "math_pipe_throttle",
          "mio_throttle", "lg_throttle", "barrier", "branch_resolving", "not_selected", "selected",
          "dispatch_stall", "drain", "tex_throttle", "membar", "sleeping", "imc_miss", "misc"]


def main(rep, launch=None):
    flt = [] if launch is None else ["-s", str(launch), "-c", "1"]
    # base units (ns, bytes, ...): ncu's default auto-scales each cell
    # separately (msecond next to usecond, GB next to MB on one line)
    out = subprocess.check_output(["ncu", "-i", rep, *flt, "--page", "raw", "--csv",
                                   "--print-units", "base"]).decode()
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")][:60]
        vals = {}
        for k, short in KEYS.items():
            if k in h:
                v, u = r[h.index(k)], units[h.index(k)]
                try:
                    x = float(v.replace(",", ""))
                except ValueError:
                    vals[short] = v
                    continue
                if u in ("nsecond", "ns"):
                    vals[short.replace("dur_us", "dur_ms") if short == "dur_us" else short] = f"{x / 1e6:.4f}"
                elif u in ("byte", "bytes"):
                    vals[short + "_GB"] = f"{x / 1e9:.4f}"
                else:
                    vals[short] = v
        st = {}
        for s in STALLS:
            k = f"smsp__pcsamp_warps_issue_stalled_{s}"
            if k in h:
                try:
                    st[s] = float(r[h.index(k)].replace(",", ""))
                except ValueError:
                    pass
        tot = sum(st.values()) or 1.0
        top = sorted(st.items(), key=lambda kv: -kv[1])[:5]
        print(name)
        print("   " + "  ".join(f"{k}={v}" for k, v in vals.items()))
        print("   stalls: " + "  ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top))


if __name__ == "__main__":
    main(sys.argv[1])
