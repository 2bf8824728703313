"""Summarise one kernel of an ncu --set full report into a tracked JSON.
Usage: python scripts/ncu_kernel_summary.py REPORT KERNEL_REGEX OUT.json [note]"""
import csv
import io
import json
import os
import re
import subprocess
import sys

rep, kre, out = sys.argv[1], sys.argv[2], sys.argv[3]
note = sys.argv[4] if len(sys.argv) > 4 else ""
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
hbm = float(json.load(open(os.path.join(root, "MEASURED_PEAKS.json")))["hbm_gbs"])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
        "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed"]
res = {"report": os.path.basename(rep), "note": note, "peak_hbm_gbs_measured": hbm, "kernels": {}}
for r in rows[2:]:
    nm = r[hdr.index("Kernel Name")]
    if not re.search(kre, nm):
        continue
    f = {k: float(r[hdr.index(k)].replace(",", "")) for k in want if k in hdr and r[hdr.index(k)]}
    if "gpu__time_duration.sum" in f:
        t_us = f["gpu__time_duration.sum"] / 1e3 if f["gpu__time_duration.sum"] > 1e5 else f["gpu__time_duration.sum"]
        mb = f.get("dram__bytes_read.sum", 0) + f.get("dram__bytes_write.sum", 0)
    stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(r[i].replace(",", ""))
              for i, k in enumerate(hdr) if k.startswith("smsp__pcsamp_warps_issue_stalled") and not
              k.endswith("not_issued") and r[i]}
    f["top_stalls_samples"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:6])
    res["kernels"][nm] = f
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1)[:2500])
