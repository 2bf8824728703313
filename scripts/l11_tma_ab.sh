# K3b A/B: TMA strips (default) vs the cp.async / LSU hybrid (MP_L1_TMA=0) on config 3, then the l1 GPU tests
mkdir -p gpurun_out
for t in 0 1 0 1; do
  echo "MP_L1_TMA=$t"
  MP_L1_TMA=$t N=4096 M=16384 Q=1 DIST=normal RELS=0.05 python scripts/timeline.py | grep -E "K3 span"
done > gpurun_out/tma_ab.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "l11 or config3 or fuzz or guard or inplace or graph" > gpurun_out/pytest_tma.log 2>&1; echo pytest=$?
