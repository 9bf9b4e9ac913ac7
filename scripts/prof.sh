# usage: bash scripts/prof.sh <tag> <clips>   -- bench timing + one ncu --set full capture of K3 fast
TAG=${1:-x}; CL=${2:-2}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 600 python bench.py --clips 32 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$TAG.log 2>&1; tail -c 1500 gpurun_out/bench_$TAG.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:resize_fast_kernel -c 1 -o gpurun_out/prof_$TAG python bench.py --clips $CL --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$TAG.log 2>&1; echo ncu=$?
