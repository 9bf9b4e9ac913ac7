VARS="ab_old ab_new" bash scripts/ab_files.sh
python paper_2604_16893_b200/_build.py -f > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_pixels.py -x -q -k "team or cfg2 or straddle or rank_shards or bands or random or mixed or cfg1" > gpurun_out/pytest_px.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_px.log
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-dedup --clips 64 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for k,v in d['side_lines'].items(): print(k, v['src'], 'k3 %.3f ms frac %.3f' % (v['k3_ms'], v['k3_frac']), v['variants'])"
