# usage: bash scripts/exp3.sh "<flags1>" "<flags2>" ...  -- 64-clip bench per nvcc flag set (experiments only)
for e in "$@"; do
  VP_EXTRA_NVCC_FLAGS="$e" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo "build failed: $e"; continue; }
  timeout 600 python bench.py --clips 64 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/exp3.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/exp3.log').read().strip().splitlines()[-1]);print('[$e]','ms',round(d['ms_per_step'],3))" || tail -3 gpurun_out/exp3.log
done
