# usage: bash scripts/gpu_round.sh [pytest-k-expr] [bench args...]
K="${1:-}"
shift || true
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv,noheader
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -3 gpurun_out/smoke.log
if [ -n "$K" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/pytest.log 2>&1; echo pytest=$?
  tail -25 gpurun_out/pytest.log
fi
if [ "$#" -gt 0 ]; then
  timeout 900 python bench.py "$@" > gpurun_out/bench.log 2>&1; echo bench=$?
  tail -c 3000 gpurun_out/bench.log
fi
