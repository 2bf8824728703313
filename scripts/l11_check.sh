# K3b iteration: timelines on the l_{1,1} shapes, then the GPU tests.
mkdir -p gpurun_out
TAG=${1:-x}
for shp in "4096 16384" "1000 16384" "6000 8192" "256 65536"; do
  set -- $shp
  N=$1 M=$2 Q=1 DIST=normal RELS=0.05 python scripts/timeline.py
done > gpurun_out/l11_tl_$TAG.log 2>&1
DT=float64 N=4096 M=16384 Q=1 DIST=normal RELS=0.05 python scripts/timeline.py >> gpurun_out/l11_tl_$TAG.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_$TAG.log 2>&1; echo pytest=$?
