"""Summarise an ncu report (--set full) into the metrics profiles/ records.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--sass N]
"""

import csv
import io
import subprocess
import sys

KEYS = [
    "Duration", "SM Frequency", "Elapsed Cycles", "SM Active Cycles", "Compute (SM) Throughput", "Memory Throughput",
    "DRAM Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy",
    "Issued Warp Per Scheduler", "No Eligible", "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction",
    "Avg. Active Threads Per Warp", "Avg. Not Predicated Off Threads Per Warp", "Executed Instructions",
    "Registers Per Thread", "Theoretical Occupancy", "Achieved Occupancy", "Waves Per SM", "Branch Efficiency",
    "Local Memory Spilling Requests",
]
RAW = [
    "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.sum", "sm__inst_executed_pipe_alu.sum", "sm__inst_executed_pipe_xu.sum",
    "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__bytes_write.sum.per_second",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
    "sm__inst_executed_pipe_uniform.sum", "smsp__inst_executed_pipe_fma.sum", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmalite_cycles_active.avg.pct_of_peak_sustained_active",
]


def ncu(*args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    out = ncu(rep, "--page", "details", "--csv")
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    print(f"# {rep}")
    name = None
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Kernel Name") != name:
            name = d.get("Kernel Name")
            print(f"kernel: {name}  grid {d.get('Grid Size')} block {d.get('Block Size')}")
        if d.get("Metric Name") in KEYS:
            print(f"  {d['Metric Name']:<45} {d['Metric Value']:>16} {d['Metric Unit']}")
    raw = ncu(rep, "--page", "raw", "--csv")
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) >= 3:
        hdr, units, vals = rr[0], rr[1], rr[2]
        for k in RAW:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:<62} {vals[i]:>18} {units[i]}")


if __name__ == "__main__":
    main()
