# one ncu --set full capture of the K3b kernel on config 3 (l_{1,1})
mkdir -p gpurun_out
TAG=${1:-x}
REPS=2 python scripts/run_l11.py > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_l1reg -s 1 -c 1 -o gpurun_out/prof_l11_$TAG -f python scripts/run_l11.py > gpurun_out/ncu_l11_$TAG.log 2>&1
echo ncu=$?
