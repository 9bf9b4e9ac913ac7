python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_pixels.py tests/test_gpu_plan.py -x -q > gpurun_out/pytest_c.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_c.log
bash scripts/configs.sh
