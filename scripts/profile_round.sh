# profiles for the round: ncu launch list of the bench command + one --set full capture of K3
TAG=${1:-r01}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/launches_bench_$TAG.log 2>&1; echo launches=$?
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:resize_fast_kernel -c 1 -o gpurun_out/k3full_$TAG \
  python bench.py --clips 8 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/k3full_$TAG.log 2>&1; echo full=$?
