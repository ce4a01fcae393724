"""Per-SASS-line executed instructions and stall samples of one kernel in an ncu report
(ncu --set full --import-source on), grouped into the loops of the listing.
    python scripts/ncu_sass_hot.py REPORT KERNEL_REGEX [top]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
import re
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
# the export holds every kernel of the report, each introduced by a "Kernel Name" line
heads = [i for i, l in enumerate(lines) if l.startswith('"Kernel Name"')] + [len(lines)]
pick = [k for k in range(len(heads) - 1) if re.search(kre, lines[heads[k]])][0]
block = lines[heads[pick] + 1:heads[pick + 1]]
rows = list(csv.reader(io.StringIO("\n".join(block))))
hdr = rows[0]
ia, isrc, iex, ism = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[1:]:
    if len(r) < len(hdr) or not r[ia].startswith("0x"):
        continue
    data.append((int(r[ia], 16), r[isrc].strip(), int(r[iex] or 0), int(r[ism] or 0)))
tot = sum(d[2] for d in data)
ts = sum(d[3] for d in data)
base = data[0][0]
print(f"kernel {kre}: {tot} warp instructions executed, {ts} stall samples")
# cumulative by 0x100-byte windows
win = {}
for a, s, e, m in data:
    k = (a - base) // 0x400
    w = win.setdefault(k, [0, 0, s])
    w[0] += e
    w[1] += m
print("by 1 KB code window (offset: instr share, stall share, first instruction)")
for k, (e, m, s) in sorted(win.items()):
    if e / tot > 0.005 or m / max(ts, 1) > 0.005:
        print(f"  +0x{k * 0x400:05x}: {100 * e / tot:5.1f}%  {100 * m / max(ts, 1):5.1f}%  {s[:60]}")
