# launch list (cold, serialised) of the hot-path kernels of the default bench command; synth (setup) excluded
TAG=${1:-launches}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:^(?!.*synth)' -c 200 --csv \
  --log-file gpurun_out/$TAG.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-dedup --no-side > gpurun_out/$TAG.log 2>&1; echo ncu=$?
