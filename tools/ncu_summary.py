"""Key ncu metrics of a report (details page) + warp-stall breakdown.
usage: python tools/ncu_summary.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "Compute (SM) Throughput", "Memory Throughput",
        "DRAM Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Registers Per Thread", "Theoretical Occupancy", "Achieved Occupancy",
        "Achieved Active Warps Per SM", "Eligible Warps Per Scheduler", "No Eligible",
        "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp", "Executed Instructions",
        "Block Limit Registers", "Block Limit Shared Mem", "Static Shared Memory Per Block",
        "Branch Efficiency", "L2 Hit Rate", "Mem Busy"]
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
im, iv, iu = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
seen = {}
for r in rows[1:]:
    if len(r) > iv and r[im] in KEYS and r[im] not in seen:
        seen[r[im]] = f"{r[iv]} {r[iu]}"
for k in KEYS:
    if k in seen:
        print(f"{k:40s} {seen[k]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
names, units, vals = rr[0], rr[1], rr[2]
stalls = []
for n, v in zip(names, vals):
    if n.startswith("smsp__average_warp_latency_issue_stalled_") or n.startswith("smsp__average_warps_issue_stalled_"):
        if n.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(v.replace(",", "")), n))
            except ValueError:
                pass
print("warp stall reasons (cycles per issued instruction):")
for v, n in sorted(stalls, reverse=True)[:12]:
    print(f"  {v:8.3f}  {n.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}")
for n, v in zip(names, vals):
    if n in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
             "sm__inst_executed_pipe_fma.sum", "sm__inst_executed_pipe_alu.sum", "sm__inst_executed_pipe_xu.sum",
             "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.sum",
             "smsp__inst_executed_op_shared_ld.sum", "lts__t_sectors_op_red.sum", "lts__t_sectors_op_atom.sum",
             "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
             "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
             "l1tex__m_l1tex2xbar_write_sectors_mem_global_op_red.sum",
             "l1tex__m_l1tex2xbar_write_sectors_mem_global_op_atom.sum",
             "SM_A.TriageCompute.sm__inst_executed_pipe_xu_realtime.avg.pct_of_peak_sustained_elapsed",
             "smsp__thread_inst_executed_per_inst_executed.ratio"):
        print(f"{n:70s} {v}")
