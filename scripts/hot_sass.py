"""Print the hottest SASS region(s) of an ncu source page (csv): address, exec count, stall samples, instruction."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, iss, ie = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
thr = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
lo = int(sys.argv[3], 16) if len(sys.argv) > 3 else 0
hi = int(sys.argv[4], 16) if len(sys.argv) > 4 else 1 << 62
base = int(rows[2][ia], 16)
for r in rows[2:]:
    try:
        a = int(r[ia], 16) - base
        n = int(r[ie])
    except ValueError:
        continue
    if n >= thr and lo <= a <= hi:
        print(f"{a:6x} {n:9d} {r[iss]:>6s}  {r[isrc].strip()}")
