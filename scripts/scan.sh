python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for c in 64 128 256 512; do
  timeout 600 python bench.py --clips $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/scan_$c.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/scan_$c.log').read().strip().splitlines()[-1]);print($c, round(d['ms_per_step'],2), round(d['ms_per_step']/$c,4), round(d['roofline']['achieved'],1))"
done
