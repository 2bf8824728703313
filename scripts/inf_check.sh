# l_inf pipeline iteration: config timelines + device config table + GPU tests
mkdir -p gpurun_out
TAG=${1:-x}
{ RELS=0.001,0.5 python scripts/timeline.py; N=1000 M=1000 DIST=normal RELS=0.1 python scripts/timeline.py;
  N=65536 M=256 RELS=0.05 python scripts/timeline.py; } > gpurun_out/inf_tl_$TAG.log 2>&1
CPU=0 timeout 900 python scripts/bench_configs.py > gpurun_out/inf_cfg_$TAG.json 2>&1; echo cfg=$?
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_$TAG.log 2>&1; echo pytest=$?
