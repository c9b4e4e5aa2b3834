#!/usr/bin/env python3
"""Summarise the ptxas logs of the build (csrc/ptxas_a0/a1/a2.log: the fp32, bf16 and fp16
units; ptxas_conv.log): registers and spill bytes per kernel (demangled).
    python tools/spills.py [substring] [--spills]"""
import glob
import re
import subprocess
import sys

log = []
for f in sorted(glob.glob("paper_1711_07240_b200/csrc/ptxas_*.log")):
    log += open(f).read().splitlines()
args = [a for a in sys.argv[1:] if not a.startswith("--")]
only_spills = "--spills" in sys.argv
flt = args[0] if args else ""
cur = None
rows = []
for line in log:
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        cur = {"name": m.group(1), "spill": 0, "regs": 0}
        rows.append(cur)
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores", line)
    if m:
        cur["spill"] = int(m.group(1))
    m = re.search(r"Used (\d+) registers", line)
    if m:
        cur["regs"] = int(m.group(1))
names = subprocess.run(["c++filt"], input="\n".join(r["name"] for r in rows), text=True,
                       capture_output=True).stdout.splitlines()
for r, n in zip(rows, names):
    n = n.replace("(anonymous namespace)::", "")
    n = n.split("(")[0]
    if flt in n and (r["spill"] or not only_spills):
        print(f"{r['regs']:4d} regs {r['spill']:4d} B spill  {n}")
