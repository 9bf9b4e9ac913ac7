python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cp paper_2604_16893_b200/libvp.so /tmp/libvp_new.so
for v in new committed new committed; do
  if [ $v = new ]; then cp /tmp/libvp_new.so paper_2604_16893_b200/libvp.so; else cp libvp_committed.so paper_2604_16893_b200/libvp.so; fi
  touch paper_2604_16893_b200/libvp.so
  timeout 600 python bench.py --clips 64 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('$v','ms',round(d['ms_per_step'],3))" || tail -3 gpurun_out/ab.log
done
