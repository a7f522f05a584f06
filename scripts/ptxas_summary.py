"""Summarise a ptxas -v log: registers and spills per (demangled) kernel.
usage: python scripts/ptxas_summary.py build/solve_kernels.o.ptxas.log [substring]"""
import re
import subprocess
import sys

cur = None
out = []
for line in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        cur = [m.group(1), None, None]
        out.append(cur)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        cur[2] = f"spill {m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        cur[1] = int(m.group(1))
names = subprocess.run(["c++filt"], input="\n".join(o[0] for o in out), capture_output=True, text=True).stdout.split("\n")
for o, nm in zip(out, names):
    if len(sys.argv) < 3 or sys.argv[2] in nm:
        print(o[1], o[2], nm[:140])
