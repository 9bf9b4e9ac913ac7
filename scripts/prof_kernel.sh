# usage: bash scripts/prof_kernel.sh <kernel-regex> <tag> [bench args...]
K=$1; TAG=$2; shift 2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$K -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e "$@" > gpurun_out/ncu_$TAG.log 2>&1; echo ncu=$?
