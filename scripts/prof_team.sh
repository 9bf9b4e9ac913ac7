# ncu --set full capture of the K3 team kernel on a cfg5 slice (one launch), summarised in gpurun_out/
# usage: bash scripts/prof_team.sh TAG [clips]
TAG=${1:-team}
CL=${2:-74}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:resize_split --launch-skip ${SKIP:-2} -c 1 -o gpurun_out/prof_$TAG \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --clips $CL > gpurun_out/ncu_$TAG.log 2>&1; echo ncu=$?
python scripts/ncu_summary.py gpurun_out/prof_$TAG.ncu-rep $CL > gpurun_out/sum_$TAG.txt 2>&1; cat gpurun_out/sum_$TAG.txt
