"""Summarise an ncu report: key SOL metrics, stall reasons, instruction mix per row-warp."""
import csv, subprocess, sys, collections, io
rep = sys.argv[1]
norm = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
def page(p, extra=()):
    return subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra], capture_output=True, text=True).stdout
det = list(csv.reader(io.StringIO(page("details"))))
want = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Achieved Occupancy",
        "Registers Per Thread", "Warp Cycles Per Issued Instruction", "Issue Slots Busy", "Executed Ipc Active",
        "No Eligible", "Active Warps Per Scheduler", "Eligible Warps Per Scheduler", "Dynamic Shared Memory Per Block",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Mem Busy", "Max Bandwidth", "Block Limit Registers", "Block Limit Shared Mem"]
for r in det[1:]:
    if len(r) > 14 and r[12] in want:
        print(f"{r[12]:40s} {r[14]:>14s} {r[13]}")
raw = list(csv.reader(io.StringIO(page("raw"))))
h, v = raw[0], raw[2]
for k, x in zip(h, v):
    if k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
             "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
             "smsp__inst_executed.sum", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
             "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active"):
        print(f"{k:60s} {x}")
st = [(k, float(x)) for k, x in zip(h, v) if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and x.replace('.', '').isdigit()]
tot = sum(x for _, x in st) or 1
print("stalls:", ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * x / tot:.0f}%" for k, x in sorted(st, key=lambda t: -t[1])[:8]))
src = list(csv.reader(io.StringIO(page("source", ("--print-source", "sass")))))
hdr = src[1]; ie = hdr.index("Instructions Executed")
b = collections.Counter()
for r in src[2:]:
    if r[ie].isdigit():
        t = r[1].split()
        op = t[1] if t and t[0].startswith("@") else (t[0] if t else "?")
        b[op] += int(r[ie])
tot = sum(b.values())
print(f"warp instructions: {tot}  per norm-unit: {tot / norm:.1f}")
print("  " + ", ".join(f"{op} {n / norm:.1f}" for op, n in b.most_common(24)))
