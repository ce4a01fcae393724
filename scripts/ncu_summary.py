"""Summarise an ncu report: key metrics per kernel + SASS opcode mix / stall reasons.
    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep [--sass]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
WANT = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'Compute (SM) Throughput', 'Achieved Occupancy',
        'Theoretical Occupancy', 'Registers Per Thread', 'Executed Ipc Active', 'Issue Slots Busy',
        'Eligible Warps Per Scheduler', 'Warp Cycles Per Issued Instruction', 'Grid Size', 'Block Size',
        'L2 Hit Rate', 'Executed Instructions', 'Dynamic Shared Memory Per Block']
out = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
ki, mi, vi, ui, ii = (hdr.index(x) for x in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit', 'ID'))
cur = None
for r in rows[1:]:
    if r[mi] in WANT:
        if r[ii] != cur:
            cur = r[ii]
            print(f"\n[{cur}] {r[ki][:110]}")
        print(f"   {r[mi]:38s} {r[vi]:>14s} {r[ui]}")
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
h = rr[0]
cols = [c for c in ('dram__bytes_read.sum', 'dram__bytes_write.sum', 'gpu__time_duration.sum') if c in h]
print("\nkernel, " + ", ".join(cols))
for r in rr[2:]:
    print(r[h.index('Kernel Name')][:60], [r[h.index(c)] for c in cols])
if '--sass' in sys.argv:
    for kid in range(4):
        s = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass',
                            '--launch-skip', str(kid), '--launch-count', '1'], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(s)))
        if len(rows) < 3:
            continue
        hh = rows[1]
        data = [x for x in rows[2:] if len(x) == len(hh)]
        ie, src, samp = hh.index("Instructions Executed"), hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)")

        def I(x):
            try:
                return int(x)
            except ValueError:
                return 0
        tot = sum(I(x[ie]) for x in data) or 1
        ts = sum(I(x[samp]) for x in data) or 1
        c, sm = collections.Counter(), collections.Counter()
        for x in data:
            toks = x[src].split()
            if not toks:
                continue
            op = toks[1] if toks[0].startswith('@') and len(toks) > 1 else toks[0]
            op = op.split('.')[0]
            c[op] += I(x[ie])
            sm[op] += I(x[samp])
        print(f"\n{rows[0][1][:90]}: {tot} warp-instr")
        print("  " + "  ".join(f"{op}:{v / tot * 100:.0f}%/{sm[op] / ts * 100:.0f}%" for op, v in c.most_common(16)))
        stall_cols = [k for k in hh if k.startswith('stall_')]
        st = {k: sum(I(x[hh.index(k)]) for x in data) for k in stall_cols}
        tt = sum(st.values()) or 1
        print("  stalls: " + "  ".join(f"{k[6:]}:{v / tt * 100:.0f}%" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:8]))
