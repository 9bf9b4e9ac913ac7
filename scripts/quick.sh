# quick: build + small parity tests + 64-clip bench
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_pixels.py -x -q -k "${1:-cfg1 or small or random_shapes or mild}" > gpurun_out/pytest_q.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_q.log
timeout 600 python bench.py --clips 64 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_q.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/bench_q.log').read().strip().splitlines()[-1]);print('ms',round(d['ms_per_step'],3),'Mtok/s',round(d['value']/1e6,2),'GB/s',round(d['roofline']['achieved'],1))"
