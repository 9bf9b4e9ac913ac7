for e in ""; do
  VP_EXTRA_NVCC_FLAGS="$e" python -c "from paper_2604_16893_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  timeout 600 python -m pytest tests/test_gpu_pixels.py -x -q -k "cfg1 or small or mild" > gpurun_out/exp2_pt.log 2>&1; echo "[$e] pytest=$?"
  timeout 600 python bench.py --clips 64 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/exp2.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/exp2.log').read().strip().splitlines()[-1]);print('[$e] ms',round(d['ms_per_step'],3))"
done
