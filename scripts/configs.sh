python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
for c in cfg2 cfg3 cfg4 cfg1; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/cfg_$c.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/cfg_$c.log').read().strip().splitlines()[-1]);print('$c ms',round(d['ms_per_step'],4),'k3 ms',round(d['roofline']['k3_ms'],4),'Mtok/s',round(d['value']/1e6,2),'GB/s',round(d['roofline']['achieved'],1))" || tail -5 gpurun_out/cfg_$c.log
done
