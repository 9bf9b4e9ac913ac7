# side lines (K3 fraction per workload) for two builds: default and the experiment flags in $1
for F in "" "$1"; do
  VP_EXTRA_NVCC_FLAGS="$F" python paper_2604_16893_b200/_build.py -f > /dev/null 2>&1
  echo "[$F]"
  python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-dedup --clips 16 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for k,v in d['side_lines'].items(): print(' ', k, v['src'], 'k3 %.3f ms frac %.3f' % (v['k3_ms'], v['k3_frac']), v['variants'])"
done
python paper_2604_16893_b200/_build.py -f > /dev/null 2>&1
