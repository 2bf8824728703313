"""Summarise an ncu source capture by SASS regions of equal execution count
(usage: python scripts/ncu_regions.py <report.ncu-rep> [min_share])."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.02
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
iW = hdr.index("Warp Stall Sampling (All Samples)")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ri = [hdr.index(k) for k in reasons]
seg, cur = [], None
for r in data:
    e = int(r[iE])
    if cur is None or e != cur["e"]:
        cur = {"e": e, "n": 0, "w": 0, "a": r[0][-5:], "s": r[iS][:34], "r": [0] * len(ri)}
        seg.append(cur)
    cur["n"] += e
    cur["w"] += int(r[iW])
    for j, k in enumerate(ri):
        try:
            cur["r"][j] += int(r[k])
        except ValueError:
            pass
tot = sum(x["n"] for x in seg)
totw = sum(x["w"] for x in seg)
print(f"instructions {tot}  stall samples {totw}")
for x in seg:
    if x["w"] / totw > thr or x["n"] / tot > thr:
        top = sorted(zip(reasons, x["r"]), key=lambda kv: -kv[1])[:4]
        print(f"{x['a']} execs={x['e']:>8d} instr={x['n'] / tot:6.1%} stalls={x['w'] / totw:6.1%} {x['s']:34s}",
              " ".join(f"{k[6:]}={v}" for k, v in top))
