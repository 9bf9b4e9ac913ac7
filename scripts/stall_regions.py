"""Stall reasons aggregated over instruction groups (by execution count bucket) of an ncu report.
usage: python scripts/stall_regions.py report.ncu-rep"""
import csv, subprocess, sys, io, collections
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
hi = next(i for i, x in enumerate(r) if "Instructions Executed" in x)
h = r[hi]; ie = h.index("Instructions Executed")
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
idx = {k: h.index(k) for k in reasons}
groups = collections.defaultdict(lambda: collections.Counter())
counts = collections.Counter()
for x in r[hi + 1:]:
    if len(x) <= ie or not x[ie].isdigit():
        continue
    n = int(x[ie]); key = n
    counts[key] += n
    for k in reasons:
        v = x[idx[k]]
        if v and v.replace('.', '').isdigit():
            groups[key][k] += float(v)
tot = sum(sum(g.values()) for g in groups.values())
for key, g in sorted(groups.items(), key=lambda t: -sum(t[1].values()))[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    s = sum(g.values())
    top = ", ".join(f"{k[6:]} {v / s * 100:.0f}%" for k, v in g.most_common(5))
    print(f"execs/line {key:>11d}: {s / tot * 100:5.1f}% of samples, instrs {counts[key]:>12d}: {top}")
