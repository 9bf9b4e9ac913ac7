# ncu --set full of the K3 team kernel (16 cfg5 clips) for the current build flags ($VP_EXTRA_NVCC_FLAGS), tag $1
python paper_2604_16893_b200/_build.py -f > gpurun_out/build.log 2>&1; echo build=$?
SKIP=2 bash scripts/prof_team.sh $1 16 > /dev/null 2>&1; echo prof=$?
head -22 gpurun_out/sum_$1.txt
