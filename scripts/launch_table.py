"""Per-kernel totals from an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv, collections, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.defaultdict(list)
for r in rows[1:]:
    try: agg[r[ki].split("(")[0].split("<")[0][-40:]].append(float(r[vi].replace(",", "")))
    except ValueError: pass
unit = rows[1][h.index("Metric Unit")] if len(rows) > 1 else ""
for k, v in sorted(agg.items(), key=lambda t: -sum(t[1])):
    print(f"{k:42s} n={len(v):4d} total={sum(v):12.1f} mean={sum(v)/len(v):10.1f} {unit}")
