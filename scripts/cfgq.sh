python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_pixels.py -x -q -k "identity or small or cfg1" > gpurun_out/pytest_c.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_c.log
bash scripts/configs.sh
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --config cfg2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/launches_c2.csv
