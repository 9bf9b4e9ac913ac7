"""Stall samples per SASS opcode x reason, split by kernel region (address ranges given as hex boundaries).
usage: ncu_stalls.py REPORT [TOP]"""
import csv, subprocess, io, sys, collections
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
hi = next(i for i, x in enumerate(r) if "Instructions Executed" in x)
h = r[hi]
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
idx = {k: h.index(k) for k in reasons}
num = lambda v: float(v) if v.replace('.', '').isdigit() else 0.0
agg = collections.defaultdict(collections.Counter)
tot = collections.Counter()
for x in r[hi + 1:]:
    if len(x) < len(h):
        continue
    t = x[1].split()
    op = t[1] if t and t[0].startswith("@") else (t[0] if t else "?")
    for k in reasons:
        v = num(x[idx[k]])
        agg[op][k] += v
        tot[k] += v
T = sum(tot.values())
print("reasons:", ", ".join(f"{k[6:]} {100 * v / T:.1f}%" for k, v in tot.most_common(10)))
for op, c in sorted(agg.items(), key=lambda t: -sum(t[1].values()))[:top]:
    s = sum(c.values())
    print(f"{op:32s} {100 * s / T:5.1f}%  " + ", ".join(f"{k[6:]} {100 * v / T:.1f}" for k, v in c.most_common(4)))
