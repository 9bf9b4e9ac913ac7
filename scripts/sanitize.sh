# compute-sanitizer over scripts/sanitize_run.py: summaries into gpurun_out/sanitize_*.txt
TOOLS=${TOOLS:-memcheck racecheck synccheck initcheck}
for tool in $TOOLS; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_run.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize_run OK' gpurun_out/sanitize_$tool.txt | tr '\n' ' ')"
done
# racecheck again on the verification build (every lane arrives on the V<->H retire barriers: racecheck only
# credits a thread's own mbarrier arrive, not lane 0's arrive after __syncwarp)
VP_EXTRA_NVCC_FLAGS="-DVP_ALL_LANES_ARRIVE=1" python paper_2604_16893_b200/_build.py -f > /dev/null 2>&1
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize_run.py > gpurun_out/sanitize_racecheck_allarrive.txt 2>&1
echo "racecheck(all lanes arrive) rc=$? $(grep -E 'RACECHECK SUMMARY|ERROR SUMMARY|sanitize_run OK' gpurun_out/sanitize_racecheck_allarrive.txt | tr '\n' ' ')"
python paper_2604_16893_b200/_build.py -f > /dev/null 2>&1
