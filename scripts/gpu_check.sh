#!/bin/bash
# One GPU round trip: smoke, GPU tests, bench, then ncu launch list + full capture.
# Usage (from the repo root, under gpurun): bash scripts/gpu_check.sh [tag] [pytest-args]
TAG=${1:-r}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_$TAG.log 2>&1; echo bench=$?
if [ "${NCU:-1}" = "1" ]; then
  CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
  $CMD > gpurun_out/ncu_plain_$TAG.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv \
      --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1; echo ncu_list=$?
  ncu --set full --clock-control none --import-source on -k regex:"k_apply|k_colnorm|k_outer" -s 12 -c 3 \
      -o gpurun_out/prof_$TAG -f $CMD > gpurun_out/ncu_full_$TAG.log 2>&1; echo ncu_full=$?
fi
