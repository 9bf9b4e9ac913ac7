# usage: bash scripts/iter.sh <tag> [pytest -k expr]
TAG=${1:-x}; K=${2:-"cfg1 or small or random_shapes or synth"}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_pixels.py -x -q -k "$K" > gpurun_out/pytest_$TAG.log 2>&1; echo pytest=$?; tail -4 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --clips 64 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$TAG.log 2>&1; tail -c 1200 gpurun_out/bench_$TAG.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:resize_fast_kernel -c 1 -o gpurun_out/prof_$TAG python bench.py --clips 2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$TAG.log 2>&1; echo ncu=$?
