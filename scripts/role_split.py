"""V/H warp-role split of an ncu report of resize_fast_kernel: samples, instructions and stall reasons per role
(the roles are separated by the two USETMAXREG instructions)."""
import csv, subprocess, io, collections, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
hi = next(i for i, x in enumerate(r) if "Instructions Executed" in x)
h = r[hi]; ie = h.index("Instructions Executed")
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
idx = {k: h.index(k) for k in reasons}
rows = [x for x in r[hi + 1:] if len(x) > ie and x[ie].isdigit()]
marks = [int(x[0], 16) for x in rows if 'SETMAXREG' in x[1]]
va, ha = marks[0], marks[1]
agg = collections.defaultdict(collections.Counter); ins = collections.Counter(); ops = collections.defaultdict(collections.Counter)
for x in rows:
    a = int(x[0], 16); g = "pro" if a < va else ("V" if a < ha else "H")
    n = int(x[ie]); ins[g] += n
    t = x[1].split(); op = t[1] if t and t[0].startswith('@') else (t[0] if t else '?'); ops[g][op] += n
    for k in reasons:
        v = x[idx[k]]
        if v and v.replace('.', '').isdigit(): agg[g][k] += float(v)
tot = sum(sum(c.values()) for c in agg.values())
norm = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
for g in ("V", "H"):
    c = agg[g]; s = sum(c.values())
    print(g, f"samples {s / tot * 100:.1f}%  instrs {ins[g] / norm / 1e6:.1f}M/unit :", ", ".join(f"{k[6:]} {v / s * 100:.0f}%" for k, v in c.most_common(6)))
    print("   ", ", ".join(f"{o} {n / norm / 1e6:.1f}" for o, n in ops[g].most_common(14)))
