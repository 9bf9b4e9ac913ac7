# small-kernel check: build, plan/pixel/rope parity, per-kernel launch list at cfg5, cfg5 + cfg1/cfg2 bench
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_plan.py tests/test_gpu_rope.py tests/test_gpu_pixels.py -x -q -k "not cfg3 and not cfg4 and not cfg2" > gpurun_out/pytest_s.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_s.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_s.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu=$?
python scripts/launch_table.py gpurun_out/launches_s.csv
for c in cfg5 cfg1 cfg2; do
timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/bench_$c.log').read().strip().splitlines()[-1]);print('$c ms',round(d['ms_per_step'],4),'k3 ms',round(d['roofline'].get('kernel_ms',0),4) if 'kernel_ms' in d['roofline'] else '', 'Mtok/s',round(d['value']/1e6,2),'GB/s',round(d['roofline']['achieved'],1))"
done
