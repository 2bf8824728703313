"""Per-source-line instruction counts / stall samples from an ncu report.
Usage: python scripts/ncu_lines.py REPORT KERNEL_REGEX [top]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", f"regex:{kre}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
agg = {}
seen_fn = 0
fname = "?"
for r in rows:
    if r and r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        ie = int(r[hdr.index("Instructions Executed")] or 0)
        ws = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        a = agg.setdefault((fname, int(r[0])), [0, 0, r[1]])
        a[0] += ie
        a[1] += ws
tot_i = sum(v[0] for v in agg.values())
tot_s = sum(v[1] for v in agg.values())
print(f"total instructions {tot_i}, samples {tot_s}")
print("-- by stall samples")
for (fn, ln), (ie, ws, src) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{fn[:14]:14s}{ln:5d} {ie:9d} {ws:6d}  {src.strip()[:80]}")
if len(sys.argv) > 4 and sys.argv[4] == "instr":
    print("-- by instructions")
    for (fn, ln), (ie, ws, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{fn[:14]:14s}{ln:5d} {ie:9d} {ws:6d}  {src.strip()[:80]}")
