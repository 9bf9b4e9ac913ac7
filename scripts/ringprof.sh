# ring iteration + profile: tests, 64-clip bench, ncu --set full of the ring kernel on 16 clips
bash scripts/ring.sh "$1"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:resize_ring_kernel -c 1 -o gpurun_out/prof_${2:-r} python bench.py --clips 16 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_${2:-r}.log 2>&1; echo ncu=$?
