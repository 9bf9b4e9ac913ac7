nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv,noheader
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -3 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest.log 2>&1; echo pytest=$?; tail -15 gpurun_out/pytest.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?; tail -c 2500 gpurun_out/bench.log
timeout 600 python bench.py --config cfg2 --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg2.log 2>&1; tail -c 600 gpurun_out/bench_cfg2.log
timeout 600 python bench.py --config cfg3 --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg3.log 2>&1; tail -c 600 gpurun_out/bench_cfg3.log
timeout 600 python bench.py --config cfg4 --no-e2e --no-cpu-baseline > gpurun_out/bench_cfg4.log 2>&1; tail -c 600 gpurun_out/bench_cfg4.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_b.log 2>&1; echo ncu=$?
