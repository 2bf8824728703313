# ncu capture of the pipelined K3b on config 3 (run under gpurun; 1 GPU)
TAG=${1:-p}
mkdir -p gpurun_out
REPS=2 python scripts/run_l11.py > /dev/null && \
ncu --set full --import-source on --clock-control none -k regex:${KREGEX:-k_l1pipe} -c 1 -o gpurun_out/$TAG -f env REPS=2 python scripts/run_l11.py > gpurun_out/${TAG}_ncu.log 2>&1; echo ncu=$?
