# A/B of compile-time variants on one box: bash scripts/abtest.sh "<flags A>" "<flags B>" ... (each = VP_EXTRA_NVCC_FLAGS)
# runs a 64-clip cfg5 bench per variant, twice, and prints k3_ms
for rep in ${REPS:-1}; do
for F in "$@"; do
  VP_EXTRA_NVCC_FLAGS="$F" python paper_2604_16893_b200/_build.py -f > /dev/null 2>&1 || { echo "build failed: $F"; continue; }
  R=$(python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --clips 64 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.3f ms  frac %.3f' % (d['roofline']['k3_ms'], d['roofline']['frac']))")
  echo "[$F] $R"
done
done
