# One full ncu capture of K3b on config 3 (run under gpurun; 1 GPU).  Usage: bash scripts/ncu_k3b.sh <tag> [lib]
TAG=${1:-k3b}
export MP_B200_LIB=$2
mkdir -p gpurun_out
REPS=2 python scripts/run_l11.py > /dev/null && \
ncu --set full --import-source on --clock-control none -k regex:k_l1reg -c 1 -o gpurun_out/$TAG -f env REPS=2 python scripts/run_l11.py > gpurun_out/${TAG}_ncu.log 2>&1; echo ncu=$?
