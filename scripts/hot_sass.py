"""Hottest SASS of an ncu report: per-opcode totals and the hottest lines in address order.
usage: python scripts/hot_sass.py report.ncu-rep [min_count] [opcode-filter]"""
import csv, subprocess, sys, io, collections
rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 1e6
flt = sys.argv[3] if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
hi = next(i for i, x in enumerate(r) if "Instructions Executed" in x)
h = r[hi]; ie = h.index("Instructions Executed"); isamp = h.index("Warp Stall Sampling (All Samples)")
rows = [(x[0][-5:], x[1].strip(), int(x[ie]), int(x[isamp] or 0)) for x in r[hi + 1:] if len(x) > ie and x[ie].isdigit()]
for a, s, n, smp in rows:
    if n >= thr and (flt is None or flt in s):
        print(a, f"{s[:100]:100s}", n, smp)
