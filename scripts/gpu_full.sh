nvidia-smi --query-gpu=name,clocks.sm --format=csv,noheader
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_all.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r10.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_r10.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['k3_ms'], d['roofline']['frac'], d['clocks'])"
bash scripts/launches.sh r10_launches > /dev/null 2>&1; echo launches=$?
SKIP=2 bash scripts/prof_team.sh r10 16 > /dev/null 2>&1; echo prof=$?
python scripts/ncu_stalls.py gpurun_out/prof_r10.ncu-rep > gpurun_out/r10_team_stalls.txt 2>&1
python scripts/ncu_sass_mem.py gpurun_out/prof_r10.ncu-rep 16 > gpurun_out/r10_team_sass_mem.txt 2>&1
true
