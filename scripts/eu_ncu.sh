mkdir -p gpurun_out
TAG=${1:-x}
SHAPES=4096x16384 RELS=0.1 REPS=1 python scripts/time_euclid.py > /dev/null 2>&1
SHAPES=4096x16384 RELS=0.1 REPS=1 ncu --set full --clock-control none -k regex:k_eu_sort -c 1 -o gpurun_out/prof_eu_$TAG -f python scripts/time_euclid.py > gpurun_out/ncu_eu_$TAG.log 2>&1; echo ncu=$?
