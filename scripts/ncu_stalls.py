"""Stall attribution of one kernel from an ncu source-page export (SASS view):
hot-loop vs the rest, and the top stalled instructions outside the hot loop.
    ncu -i REP --page source --csv --print-source=sass > SRC.csv
    python scripts/ncu_stalls.py SRC.csv KERNEL_INDEX [top]"""
import collections
import csv
import io
import re
import sys

lines = open(sys.argv[1]).read().splitlines()
kidx = int(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
heads = [i for i, l in enumerate(lines) if l.startswith('"Kernel Name"')] + [len(lines)]
print(lines[heads[kidx]][:140])
rows = list(csv.reader(io.StringIO("\n".join(lines[heads[kidx] + 1:heads[kidx + 1]]))))
h, R = rows[0], rows[1:]
ix = {k: h.index(k) for k in h}
st = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
ex = [int(r[ix["Instructions Executed"]] or 0) for r in R]
mx = max(ex)
hot = [r for r, e in zip(R, ex) if e >= 0.9 * mx]
cnt = lambda rs: collections.Counter({k: sum(int(r[ix[k]] or 0) for r in rs) for k in st})
ch, ca = cnt(hot), cnt(R)
th, ta = sum(ch.values()), sum(ca.values())
print(f"instructions executed: {sum(ex)}; hot loop {len(hot)} SASS x {mx}: {sum(e for e in ex if e >= 0.9 * mx) / sum(ex):.1%} of instructions, {th / ta:.1%} of stall samples")
print("hot:  ", ", ".join(f"{k[6:]}={v}" for k, v in ch.most_common(8)))
print("rest: ", ", ".join(f"{k[6:]}={ca[k] - ch[k]}" for k, _ in (ca - ch).most_common(8)))
rest = [(i, r) for i, (r, e) in enumerate(zip(R, ex)) if e < 0.9 * mx]
rest.sort(key=lambda x: -int(x[1][ix["Warp Stall Sampling (All Samples)"]] or 0))
for i, r in rest[:top]:
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    tp = sorted([(k[6:], int(r[ix[k]] or 0)) for k in st], key=lambda x: -x[1])[:2]
    print(f"  #{i:5d} {s:4d} x{r[ix['Instructions Executed']]:>7s} {r[ix['Source']].strip()[:64]:64s} {tp}")
