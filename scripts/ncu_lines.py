"""Per CUDA source line of an ncu report (mixed cuda,sass source page): instructions, shared-memory wavefronts and
stall samples, normalised per unit (e.g. per clip).  usage: ncu_lines.py REPORT NORM [TOP]"""
import csv, subprocess, io, sys, collections
rep, norm = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 50
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0, ""])
f = "?"
h = None
cur = None
for x in csv.reader(io.StringIO(out)):
    if not x:
        continue
    if x[0] == "File Path":
        f = x[1].split("/")[-1]; continue
    if x[0] == "Line No":
        h = x; ie = h.index("Instructions Executed"); iw = h.index("L1 Wavefronts Shared")
        isamp = h.index("Warp Stall Sampling (All Samples)"); continue
    if h is None or len(x) <= ie:
        continue
    if x[0]:
        cur = (f, int(x[0]))
        agg[cur][3] = x[1].strip()[:80]
    if cur is None or not x[ie].replace('.', '').isdigit():
        continue
    a = agg[cur]
    num = lambda v: float(v) if v.replace('.', '').isdigit() else 0.0
    a[0] += num(x[ie]); a[1] += num(x[iw]); a[2] += num(x[isamp])
ti = sum(a[0] for a in agg.values()); tw = sum(a[1] for a in agg.values()); ts = sum(a[2] for a in agg.values()) or 1
print(f"total: {ti / norm / 1e6:.2f}M instr, {tw / norm / 1e6:.2f}M smem wavefronts per unit")
for k, a in sorted(agg.items(), key=lambda t: -t[1][2])[:top]:
    if a[0] == 0 and a[2] == 0:
        continue
    print(f"{a[0] / norm / 1e6:6.2f}M  {a[1] / norm / 1e6:6.2f}Mwf {100 * a[2] / ts:5.1f}%  {k[0][:16]}:{k[1]:<4} {a[3]}")
