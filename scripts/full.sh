# full round check: build, smoke, all GPU tests, default bench, launch list
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_full.log 2>&1; echo pytest=$?; tail -5 gpurun_out/pytest_full.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench=$?; tail -c 2500 gpurun_out/bench_full.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref=$?; tail -c 800 gpurun_out/bench_ref.log
