for e in 0 1 2 3; do
  VP_EXTRA_NVCC_FLAGS="-DVP_EXPERIMENT=$e" python -c "from paper_2604_16893_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  timeout 600 python bench.py --clips 64 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/exp_$e.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/exp_$e.log').read().strip().splitlines()[-1]);print('exp $e ms',round(d['ms_per_step'],3))"
done
