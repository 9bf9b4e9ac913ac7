"""Shared-memory wavefronts (actual / ideal) and instruction counts per SASS opcode of an ncu report, per unit.
usage: ncu_sass_mem.py REPORT NORM"""
import csv, subprocess, io, sys, collections
rep, norm = sys.argv[1], float(sys.argv[2])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
hi = next(i for i, x in enumerate(r) if "Instructions Executed" in x)
h = r[hi]
ie, iw, iwi, isamp = (h.index(k) for k in ("Instructions Executed", "L1 Wavefronts Shared", "L1 Wavefronts Shared Ideal",
                                           "Warp Stall Sampling (All Samples)"))
num = lambda v: float(v) if v.replace('.', '').isdigit() else 0.0
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0, 0.0])
for x in r[hi + 1:]:
    if len(x) <= iwi:
        continue
    t = x[1].split()
    op = t[1] if t and t[0].startswith("@") else (t[0] if t else "?")
    a = agg[op]
    a[0] += num(x[ie]); a[1] += num(x[iw]); a[2] += num(x[iwi]); a[3] += num(x[isamp])
ts = sum(a[3] for a in agg.values()) or 1
print(f"instr {sum(a[0] for a in agg.values()) / norm / 1e6:.2f}M  smem wavefronts {sum(a[1] for a in agg.values()) / norm / 1e6:.2f}M "
      f"(ideal {sum(a[2] for a in agg.values()) / norm / 1e6:.2f}M) per unit")
for op, a in sorted(agg.items(), key=lambda t: -t[1][0])[:30]:
    print(f"{op:34s} {a[0] / norm / 1e6:7.2f}M instr  {a[1] / norm / 1e6:6.2f}M wf (ideal {a[2] / norm / 1e6:5.2f}M)  {100 * a[3] / ts:5.1f}% samples")
