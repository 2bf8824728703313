"""Summarise an ncu --csv launch list: per-kernel count, mean duration, DRAM bytes."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(list)
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        agg[(d["Kernel Name"][:70], d["Metric Name"])].append(float(d["Metric Value"].replace(",", "")))
names = sorted({k[0] for k in agg})
print(f"{'kernel':70s} {'n':>4s} {'us':>9s} {'dram_rd_MB':>11s} {'dram_wr_MB':>11s}")
for nm in names:
    t = agg.get((nm, "gpu__time_duration.sum"), [0])
    rd = agg.get((nm, "dram__bytes_read.sum"), [0])
    wr = agg.get((nm, "dram__bytes_write.sum"), [0])
    print(f"{nm:70s} {len(t):4d} {sum(t)/len(t)/1e3:9.2f} {sum(rd)/len(rd)/1e6:11.2f} {sum(wr)/len(wr)/1e6:11.2f}")
