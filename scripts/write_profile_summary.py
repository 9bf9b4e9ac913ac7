"""Write profiles/<tag>_summary.md + profiles/traffic.json from a launch-list csv and an ncu --set full report."""
import csv, collections, json, subprocess, sys, io, os
tag, launches_csv, rep, clips = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rows = list(csv.reader(open(launches_csv)))
for i, r in enumerate(rows):
    if 'Kernel Name' in r:
        hdr = r; start = i + 1; break
ki, vi, mi = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Name')
agg = collections.defaultdict(list)
for r in rows[start:]:
    if len(r) > vi and r[mi] == 'gpu__time_duration.sum':
        agg[r[ki].split('(')[0].replace('void ', '').split('::')[-1]].append(float(r[vi].replace(',', '')))
tot = sum(sum(v) for v in agg.values() if True)
hot = {k: v for k, v in agg.items() if not k.startswith('synth_kernel')}
tot_hot = sum(sum(v) for v in hot.values())
def page(p):
    return list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", p, "--csv"], capture_output=True, text=True).stdout)))
det = page("details")
want = ["Duration", "DRAM Throughput", "Compute (SM) Throughput", "Achieved Occupancy", "Registers Per Thread",
        "Issue Slots Busy", "Executed Ipc Active", "No Eligible", "Eligible Warps Per Scheduler",
        "Dynamic Shared Memory Per Block", "L2 Hit Rate", "L1/TEX Hit Rate"]
kv = {}
for r in det[1:]:
    if len(r) > 14 and r[12] in want and r[12] not in kv:
        kv[r[12]] = f"{r[14]} {r[13]}"
raw = page("raw")
h, v = raw[0], raw[2]
rawd = dict(zip(h, v))
SC = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
def nbytes(name):
    return float(rawd.get(name, "nan")) * SC.get(raw[1][h.index(name)], 1) if name in h else float("nan")
rd, wr, scale = nbytes("dram__bytes_read.sum"), nbytes("dram__bytes_write.sum"), 1
st = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(x)) for k, x in rawd.items()
      if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and x.replace('.', '').isdigit()]
stt = sum(x for _, x in st) or 1
with open(os.path.join(ROOT, "profiles", f"{tag}_summary.md"), "w") as f:
    f.write(f"# Profile summary {tag}\n\n## Launch list (ncu --metrics gpu__time_duration.sum --clock-control none, `bench.py --steps 2 --warmup 1`, cfg5 512 clips)\n\n")
    f.write("Cold-cache, serialised per-launch times: compare shares, not absolutes. synth_kernel is the untimed input generator.\n\n")
    f.write("| kernel | launches | total ms | mean us | share of hot path |\n|---|---|---|---|---|\n")
    for k, vv in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        share = f"{100 * sum(vv) / tot_hot:.2f}%" if k in hot else "(input gen)"
        f.write(f"| {k} | {len(vv)} | {sum(vv) / 1e6:.3f} | {sum(vv) / len(vv) / 1e3:.1f} | {share} |\n")
    f.write(f"\n## K3 resize_fast_kernel, `ncu --set full` ({clips} cfg5 clips, one launch)\n\n")
    for k in want:
        if k in kv:
            f.write(f"- {k}: {kv[k]}\n")
    f.write(f"- dram__bytes_read.sum: {rd * scale / 1e9:.4f} GB, dram__bytes_write.sum: {wr * scale / 1e9:.4f} GB "
            f"(per clip {(rd + wr) * scale / clips / 1e9:.4f} GB; algorithmic per clip 0.2760 GB)\n")
    f.write("- stall reasons (pc sampling): " + ", ".join(f"{k} {100 * x / stt:.0f}%" for k, x in sorted(st, key=lambda t: -t[1])[:8]) + "\n")
with open(os.path.join(ROOT, "profiles", "traffic.json"), "w") as f:
    json.dump({"k3_dram_bytes_per_clip": (rd + wr) * scale / clips, "source": f"profiles/{tag}_summary.md",
               "report_clips": clips, "read_bytes": rd * scale, "write_bytes": wr * scale}, f, indent=1)
print(open(os.path.join(ROOT, "profiles", f"{tag}_summary.md")).read())
