"""Register / stack usage of the kernels in libmp_b200.so matching a regex (cuobjdump)."""
import re
import subprocess
import sys
pat = re.compile(sys.argv[1] if len(sys.argv) > 1 else ".")
out = subprocess.run("cuobjdump --dump-resource-usage paper_2405_02086_b200/libmp_b200.so | c++filt", shell=True,
                     capture_output=True, text=True).stdout.splitlines()
name = None
for ln in out:
    m = re.search(r"Function (.*):", ln)
    if m:
        name = m.group(1)
        continue
    r = re.search(r"REG:(\d+) STACK:(\d+)", ln)
    if r and name and pat.search(name):
        print(f"REG {r.group(1):>3} STACK {r.group(2):>4}  {name.split('(')[0]}")
