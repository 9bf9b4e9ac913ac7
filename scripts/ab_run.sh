# same-box A/B of ab_old/ vs ab_new/ (64-clip cfg5 K3) + the K3 parity subset on the new tree
VARS="ab_old ab_new" bash scripts/ab_files.sh
python paper_2604_16893_b200/_build.py -f > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_pixels.py -x -q -k "${K:-team or cfg2 or straddle or rank_shards or bands or random or mixed or cfg5_bench}" > gpurun_out/pytest_px.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_px.log
