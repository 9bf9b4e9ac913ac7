# same-box A/B of compile-time K3 variants (experiments): 64-clip cfg5 K3 time per flag set
python paper_2604_16893_b200/_build.py -f > /dev/null 2>&1
REPS="1 2" bash scripts/abtest.sh "" "-DVP_WIDE_VPX=2" "-DVP_WIDE_VPX=2 -DVP_WIDE2_VREGS=64 -DVP_WIDE2_HREGS=64"
python paper_2604_16893_b200/_build.py -f > /dev/null 2>&1
VP_EXTRA_NVCC_FLAGS="-DVP_WIDE_VPX=2" python paper_2604_16893_b200/_build.py -f > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_pixels.py -q -x -k "team or cfg2 or straddle or random or cfg5_bench" 2>&1 | tail -2
python paper_2604_16893_b200/_build.py -f > /dev/null 2>&1
