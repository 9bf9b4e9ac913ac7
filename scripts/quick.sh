python paper_2604_16893_b200/_build.py -f > /dev/null
python -m pytest tests/test_gpu_pixels.py -x -q -k "team or cfg2 or cfg1 or small_mixed or straddle or random or cfg4" 2>&1 | tail -2
bash scripts/abtest.sh "" "-DVP_TEAM_HINT=200" "-DVP_TEAM_HINT=2000"
