"""Turn an ncu round capture (gpurun_out/) into the tracked summaries under profiles/.
Usage: python scripts/profile_summary.py <tag> [<round-name>]"""
import collections
import csv
import io
import json
import os
import shutil
import subprocess
import sys

tag = sys.argv[1]
name = sys.argv[2] if len(sys.argv) > 2 else tag
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
go = os.path.join(root, "gpurun_out")
prof = os.path.join(root, "profiles")
os.makedirs(prof, exist_ok=True)
peaks = json.load(open(os.path.join(root, "MEASURED_PEAKS.json")))
hbm = float(peaks["hbm_gbs"])


def launch_table(path):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, collections.defaultdict(list)
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            agg[(d["Kernel Name"], d["Metric Name"])].append(float(d["Metric Value"].replace(",", "")))
    out = {}
    for nm in sorted({k[0] for k in agg}):
        t = agg.get((nm, "gpu__time_duration.sum"), [0])
        rd = agg.get((nm, "dram__bytes_read.sum"), [0])
        wr = agg.get((nm, "dram__bytes_write.sum"), [0])
        out[nm] = {"launches": len(t), "avg_us": sum(t) / len(t) / 1e3, "dram_read_MB": sum(rd) / len(rd) / 1e6,
                   "dram_write_MB": sum(wr) / len(wr) / 1e6}
    return out


summary = {"tag": tag, "peak_hbm_gbs_measured": hbm, "command": "python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"}
for kind, fn in (("launches_cold_cache", f"launches_{tag}.csv"), ("launches_no_cache_control", f"launches_nocache_{tag}.csv")):
    p = os.path.join(go, fn)
    if os.path.exists(p):
        summary[kind] = launch_table(p)
        shutil.copy(p, os.path.join(prof, f"{name}_{fn.replace('_' + tag, '')}"))
rep = os.path.join(go, f"prof_{tag}.ncu-rep")
if os.path.exists(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
            "launch__registers_per_thread", "launch__occupancy_limit_registers",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
            "smsp__inst_executed.sum", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
            "dram__cycles_active.avg.pct_of_peak_sustained_elapsed"]
    full = {}
    for r in rows[2:]:
        nm = r[hdr.index("Kernel Name")]
        full[nm] = {k: float(r[hdr.index(k)].replace(",", "")) for k in want if k in hdr and r[hdr.index(k)]}
        f = full[nm]
        if "gpu__time_duration.sum" in f:
            mb = f.get("dram__bytes_read.sum", 0) + f.get("dram__bytes_write.sum", 0)
            f["dram_GBps"] = mb / (f["gpu__time_duration.sum"] * 1e-6) / 1e3
            f["dram_frac_of_measured_peak"] = f["dram_GBps"] / hbm
    summary["full_set"] = full
    for nm, f in full.items():
        if "k_apply" in nm:
            traffic = (f.get("dram__bytes_read.sum", 0) + f.get("dram__bytes_write.sum", 0)) * 1e6
            json.dump({"kernel": nm, "bytes_per_launch": traffic, "source": f"ncu --set full ({name})",
                       "note": "cold-cache replay (ncu flushes caches): the in-pipeline L2 reuse is not visible here"},
                      open(os.path.join(prof, "k3_traffic.json"), "w"), indent=1)
json.dump(summary, open(os.path.join(prof, f"{name}_ncu_summary.json"), "w"), indent=1)
print(json.dumps(summary, indent=1)[:3000])
