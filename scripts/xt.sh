# same-box A/B of compile-time K3 variants (experiments): 64-clip cfg5 K3 time per flag set
REPS="1" bash scripts/abtest.sh "" "-Xptxas --allow-expensive-optimizations=true" "-Xptxas -O2" "-DVP_TEAM_HINT=200" "-Xptxas -O3 -Xptxas --extra-device-vectorization"
python paper_2604_16893_b200/_build.py -f > /dev/null 2>&1
