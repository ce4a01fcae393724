"""Print registers / spills per kernel from the ptxas logs: python scripts/regs.py [substring]"""
import glob
import re
import subprocess
import sys

pat = sys.argv[1] if len(sys.argv) > 1 else ""
for f in sorted(glob.glob("paper_2302_02390_b200/_build/*.ptxas.log")):
    cur, sp = None, "0"
    for line in open(f):
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
            continue
        m = re.search(r"(\d+) bytes spill stores", line)
        if m:
            sp = m.group(1)
            continue
        m = re.search(r"Used (\d+) registers", line)
        if m and cur and pat in cur:
            print(f"{m.group(1):>4} regs  spill {sp:>3}  {cur.replace('void qsdp::', '')[:110]}")
