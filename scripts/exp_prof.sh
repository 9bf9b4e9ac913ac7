# usage: bash scripts/exp_prof.sh "<nvcc flags>" <tag>  -- ncu --set full of resize_fast_kernel (16 clips) for an experiment build
VP_EXTRA_NVCC_FLAGS="$1" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 900 ncu --set full --import-source on --clock-control none -k regex:resize_fast_kernel -c 1 -o gpurun_out/prof_$2 python bench.py --clips 16 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$2.log 2>&1; echo ncu=$?
