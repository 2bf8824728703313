mkdir -p gpurun_out
N=4096 M=16384 Q=1 DIST=normal RELS=0.05 python scripts/timeline.py > gpurun_out/l11_tl.log 2>&1
N=1000 M=16384 Q=1 DIST=normal RELS=0.05 python scripts/timeline.py >> gpurun_out/l11_tl.log 2>&1
N=6000 M=8192 Q=1 DIST=normal RELS=0.05 python scripts/timeline.py >> gpurun_out/l11_tl.log 2>&1
REPS=2 python scripts/run_l11.py > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_l1reg -s 1 -c 1 -o gpurun_out/prof_l11b -f python scripts/run_l11.py > gpurun_out/ncu_l11b.log 2>&1
echo done
