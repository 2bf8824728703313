#!/bin/bash
# ncu evidence for the headline bench (run under gpurun; 1 GPU).
# Usage: bash scripts/profile_round.sh <tag>
TAG=${1:-r1}
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/prof_plain_$TAG.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1; echo ncu_list=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_nocache_$TAG.csv $CMD > gpurun_out/ncu_launch_nc_$TAG.log 2>&1; echo ncu_list_nocache=$?
ncu --set full --clock-control none --import-source on -k regex:"k_apply|k_colnorm|k_outer" -s 6 -c 3 \
    -o gpurun_out/prof_$TAG -f $CMD > gpurun_out/ncu_full_$TAG.log 2>&1; echo ncu_full=$?
