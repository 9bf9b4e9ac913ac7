# K3 ring iteration: build, ring parity tests (+ extra -k expr), 64-clip bench
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_pixels.py -x -q -k "${1:-ring or cfg2_one or cfg1 or small}" > gpurun_out/pytest_ring.log 2>&1; echo pytest=$?; tail -30 gpurun_out/pytest_ring.log | grep -v "^$" | tail -25
timeout 600 python bench.py --clips 64 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_ring.log 2>&1; echo bench=$?
python -c "import json;d=json.loads(open('gpurun_out/bench_ring.log').read().strip().splitlines()[-1]);print('ms',round(d['ms_per_step'],3),'Mtok/s',round(d['value']/1e6,2),'GB/s',round(d['roofline']['achieved'],1), 'frac', round(d['roofline']['frac'],3))" || tail -20 gpurun_out/bench_ring.log
