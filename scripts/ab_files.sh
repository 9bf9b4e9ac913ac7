# same-box A/B of two source trees of the K3 files (ab_old/ vs ab_new/), 64-clip cfg5 K3 time, twice each
B=paper_2604_16893_b200/csrc
for rep in 1 2; do for v in ${VARS:-ab_old ab_new}; do
  cp $v/* $B/; python paper_2604_16893_b200/_build.py -f > /dev/null 2>&1 || echo "build failed $v"
  R=$(python bench.py --steps 8 --warmup 3 --no-e2e --no-cpu-baseline --no-dedup --no-side --clips ${CLIPS:-64} 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.3f ms  frac %.3f' % (d['roofline']['k3_ms'], d['roofline']['frac']))")
  echo "[$v] $R"
done; done
cp ab_new/* $B/
