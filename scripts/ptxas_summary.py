"""Registers / spills per kernel from the build's ptxas -v logs (paper_2302_02390_b200/_build/*.ptxas.log).
    python scripts/ptxas_summary.py [regex]"""
import glob
import os
import re
import subprocess
import sys

pat = re.compile(sys.argv[1]) if len(sys.argv) > 1 else None
root = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2302_02390_b200", os.environ.get("QSDP_BUILD", "_build"))
for log in sorted(glob.glob(os.path.join(root, "*.ptxas.log"))):
    name, spill = None, (0, 0)
    for line in open(log):
        m = re.search(r"Compiling entry function '(\S+)'", line) or re.search(r"Function properties for (\S+)", line)
        if m:
            name = m.group(1)
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and name:
            spill = (int(m.group(2)), int(m.group(3)))
        m = re.search(r"Used (\d+) registers", line)
        if m and name:
            dn = subprocess.run(["c++filt"], input=name, capture_output=True, text=True).stdout.strip()
            if pat is None or pat.search(dn):
                print(f"{os.path.basename(log)[:-10]:16s} regs {m.group(1):>4s} spill {spill}  {dn[:110]}")
            name = None
