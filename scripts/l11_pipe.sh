# K3b pipelined strips: config-3 timeline (f32, f64) + the l1 GPU tests.
mkdir -p gpurun_out
TAG=${1:-x}
{
N=4096 M=16384 Q=1 DIST=normal RELS=0.05 python scripts/timeline.py
DT=float64 N=4096 M=16384 Q=1 DIST=normal RELS=0.05 python scripts/timeline.py
N=3000 M=16384 Q=1 DIST=normal RELS=0.05 python scripts/timeline.py
} > gpurun_out/l11_tl_$TAG.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "${PYTEST_K:-l1 or config3 or guard or fuzz or nonfinite}" > gpurun_out/pytest_$TAG.log 2>&1; echo pytest=$?
