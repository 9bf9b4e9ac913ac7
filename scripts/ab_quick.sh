# quick same-box check: build, a K3 parity subset, 64-clip and 512-clip cfg5 K3 times
nvidia-smi --query-gpu=name,clocks.sm --format=csv,noheader
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_pixels.py -x -q -k "${K:-team or cfg2 or straddle or cfg5_bench}" > gpurun_out/pytest_px.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_px.log
for r in 1 2; do python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-dedup --no-side --clips 64 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('64 clips: %.3f ms frac %.3f' % (d['roofline']['k3_ms'], d['roofline']['frac']))"; done
[ -n "$FULL" ] && python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-dedup --no-side 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('512 clips: %.3f ms frac %.3f' % (d['roofline']['k3_ms'], d['roofline']['frac']))"
true
