# same-box A/B of compile-time K3 variants (experiments): 64-clip cfg5 K3 time per flag set
REPS="1" bash scripts/abtest.sh "" "-DVP_TEAM_GRP=16 -DVP_TEAM_DEPTH=32" "-DVP_TEAM_DEPTH=24" "-DVP_TEAM_GRP=4 -DVP_TEAM_DEPTH=16"
python paper_2604_16893_b200/_build.py -f > /dev/null 2>&1
