# Per-kernel ncu inventory over the five configs + K2 cooperative + euclid +
# the generic multi-level chain (run under gpurun, one GPU).  Cold cache
# (ncu's default cache control), every kernel of every case; the summary keeps
# the last launch of each kernel.  Writes gpurun_out/inv_<case>.csv + .log.
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__block_size,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
for c in ${CASES:-c1 c2 c2_f64 c3_l11 c3_l11_f64 c3_l12 c4 ml111 c5 k2_coop euclid}; do
  CASE=$c python scripts/kernel_cases.py > gpurun_out/inv_$c.plain 2>&1 || { echo "$c plain failed"; continue; }
  CASE=$c ncu --metrics $M --clock-control none --csv --log-file gpurun_out/inv_$c.csv \
      python scripts/kernel_cases.py > gpurun_out/inv_$c.log 2>&1
  echo "$c ncu=$?"
done
