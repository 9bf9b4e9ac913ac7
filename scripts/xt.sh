# same-box A/B of compile-time K3 variants (experiments): 64-clip cfg5 K3 time per flag set
REPS="1 2" bash scripts/abtest.sh "" "-DVP_EXP_NOCVTAHEAD"
python paper_2604_16893_b200/_build.py -f > /dev/null 2>&1
