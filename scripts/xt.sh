python paper_2604_16893_b200/_build.py -f > /dev/null 2>&1 || echo BUILD FAIL
timeout 600 python -m pytest tests/test_gpu_pixels.py -x -q -k "team or cfg1 or small_mixed or random or cfg2 or straddle" 2>&1 | tail -2
REPS="1 2" bash scripts/abtest.sh "" "-DXT_NOV=1" "-DXT_NOH=1"
