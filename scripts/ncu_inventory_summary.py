"""Summarise scripts/ncu_inventory.sh output into profiles/r2_kernels.json:
for every kernel of every case (last launch): ncu time, DRAM bytes read /
written, the algorithmic bytes of that kernel (SURVEY §8d per-unit figures x
the case's shape), achieved algorithmic GB/s and its fraction of the
measured HBM peak, plus occupancy / issue figures."""
import collections
import csv
import json
import os
import re
import sys

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
go = os.path.join(root, "gpurun_out")
peak = float(json.load(open(os.path.join(root, "MEASURED_PEAKS.json")))["hbm_gbs"])


def algo_bytes(kernel, meta):
    """Algorithmic bytes of one launch (None for latency-bound kernels)."""
    n, m, s, fs = meta["n"], meta["m"], meta["s"], meta.get("f_surv", 1.0)
    N = n * m
    if "k_colnorm_finalize" in kernel or "k_colnorm_reduce" in kernel:
        return None
    if "k_colnorm" in kernel:
        return s * N  # one read
    if "k_apply" in kernel:
        return s * N * (1.0 + fs)  # surviving reads + full write
    if re.search(r"k_l1(reg|quad|cols|strip)", kernel):
        return 2.0 * s * N  # strip read + write
    if "k_perturb" in kernel:
        return 2.0 * s * N
    if "k_eu_gather" in kernel:
        return 2.0 * s * N
    if "k_eu_sort" in kernel:
        return None  # compute-bound (shared memory)
    return None


out = {"peak_hbm_gbs": peak, "peak_source": "MEASURED_PEAKS.json hbm_gbs",
       "method": "ncu --metrics ... --clock-control none (default cache control: caches flushed before each "
                 "kernel, i.e. cold), scripts/ncu_inventory.sh; last launch of each kernel per case",
       "cases": {}}
for fn in sorted(os.listdir(go)):
    mt = re.match(r"inv_(.+)\.csv$", fn)
    if not mt:
        continue
    case = mt.group(1)
    meta = None
    for line in open(os.path.join(go, f"inv_{case}.log"), errors="replace"):
        if line.startswith("META "):
            meta = json.loads(line[5:])
    if meta is None:
        continue
    rows = list(csv.reader(open(os.path.join(go, fn))))
    hdr = None
    last = collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        name = d["Kernel Name"]
        if not re.search(r"k_[a-z]", name) or "at::" in name:
            continue
        key = re.sub(r"\(.*", "", name).strip()
        last.setdefault(key, {})
        # later launches overwrite: the last launch wins
        if d["Metric Name"] in last[key] and d["ID"] != last[key].get("_id"):
            last[key] = {}
        last[key]["_id"] = d["ID"]
        last[key]["_name"] = name
        last[key][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    kern = {}
    for key, v in last.items():
        t_us = v.get("gpu__time_duration.sum", 0.0) / 1e3
        km = meta
        if meta["case"] == "ml111" and "<double" in v["_name"]:
            # the generic chain's level-1 kernels run on the 256 x 256 f64 norm array
            km = dict(meta, n=256, m=256, s=8)
        ab = algo_bytes(v["_name"], km)
        e = {"time_us": round(t_us, 2),
             "dram_read_MB": round(v.get("dram__bytes_read.sum", 0) / 1e6, 2),
             "dram_write_MB": round(v.get("dram__bytes_write.sum", 0) / 1e6, 2),
             "dram_throughput_pct": v.get("dram__throughput.avg.pct_of_peak_sustained_elapsed"),
             "grid": v.get("launch__grid_size"), "block": v.get("launch__block_size"),
             "regs": v.get("launch__registers_per_thread"),
             "warps_active_pct": v.get("sm__warps_active.avg.pct_of_peak_sustained_active"),
             "issue_active_pct": v.get("smsp__issue_active.avg.pct_of_peak_sustained_active")}
        if ab is not None and t_us > 0:
            gbs = ab / (t_us * 1e-6) / 1e9
            e.update({"algorithmic_MB": round(ab / 1e6, 2), "achieved_GBs": round(gbs, 1),
                      "frac_of_peak": round(gbs / peak, 3),
                      "traffic_over_algorithmic": round((v.get("dram__bytes_read.sum", 0) +
                                                         v.get("dram__bytes_write.sum", 0)) / ab, 3)})
        kern[key] = e
    out["cases"][case] = {"meta": meta, "kernels": kern}
dst = sys.argv[1] if len(sys.argv) > 1 else os.path.join(root, "profiles", "r2_kernels.json")
json.dump(out, open(dst, "w"), indent=1)
for c, d in out["cases"].items():
    print(c, d["meta"])
    for k, e in d["kernels"].items():
        print(f"   {k[:70]:70s} {e['time_us']:9.1f} us  rd {e['dram_read_MB']:8.1f} wr {e['dram_write_MB']:8.1f} MB"
              + (f"  {e['achieved_GBs']:7.0f} GB/s {e['frac_of_peak']:.3f}" if "achieved_GBs" in e else ""))
