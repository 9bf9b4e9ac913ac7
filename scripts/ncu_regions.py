"""Stall samples per code region (V loop vs H loop vs spin waits) from an ncu source page."""
import csv, subprocess, sys, io, collections
rep = sys.argv[1]
src = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                                                  capture_output=True, text=True).stdout)))
hdr = src[1]; data = src[2:]
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ci = {c: hdr.index(c) for c in cols}
ie = hdr.index("Instructions Executed")
# classify instructions by the nearest preceding marker: FFMA2 with .F32 on 6 pairs => V ring; LDS.128 => H
region = "prologue"; agg = collections.defaultdict(collections.Counter); ins = collections.Counter()
for r in data:
    t = r[1]
    if "I2F.U8" in t: region = "V"
    elif "LDS.128" in t: region = "H"
    elif "TRYWAIT" in t: region = region.split("+")[0] + "+wait"
    for c in cols:
        v = r[ci[c]]
        if v.isdigit(): agg[region][c] += int(v)
    if r[ie].isdigit(): ins[region] += int(r[ie])
for reg, cnt in agg.items():
    tot = sum(cnt.values())
    print(f"{reg:12s} samples {tot:8d} instr {ins[reg]:11d}  " + ", ".join(f"{k[6:]} {100*v/max(tot,1):.0f}%" for k, v in cnt.most_common(5)))
