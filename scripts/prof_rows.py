"""Launch each §8(f) kernel once on a GPT-2 wte-sized segment (38.6 M fp32) for
an ncu capture: levels quantize (LQ) / dequantize (LD), wire encode / decode,
K4 + lattice step, and the 2-source K4 (multi-source fast path).

    ncu --set full -k "regex:levels|wire|lat_fast|dequant_kernel" -c 8 python scripts/prof_rows.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_02390_b200.lattice import LatticeStep, dequant_accumulate_lattice, shift_key  # noqa: E402
from paper_2302_02390_b200.levels import LevelTable, dequantize_levels, learn_levels, quantize_levels  # noqa: E402
from paper_2302_02390_b200.quantize import QuantSpec, SegmentKey, dequant_accumulate, quantize_segments  # noqa: E402
from paper_2302_02390_b200.wire import decode_kernels, encode_segment  # noqa: E402

n = 38633472
dev = torch.device("cuda", 0)
x = torch.randn(n, device=dev) * 0.02
g = torch.randn(n, device=dev) * 1e-3
table = learn_levels(torch.rand(1 << 16, device=dev, dtype=torch.float64), LevelTable.uniform(8))
ls = QuantSpec(8, 1024, "levels")
lc, lm = quantize_levels(x, ls, table)                                   # LQ
dequantize_levels(lc, lm, n, ls, table, dtype=torch.float32)              # LD
ws = QuantSpec(8, 1024, "shift")
(wc, wm), = quantize_segments([(x, 0, SegmentKey(0, 1, 0, 0, 0))], ws)
msg = encode_segment(wc, wm, n, ws)                                        # wire encode
decode_kernels([msg])()                                                    # wire decode
gs = QuantSpec(8, 1024, "uniform_stochastic")
(g0c, g0m), (g1c, g1m) = quantize_segments([(g, 0, SegmentKey(0, 1, 0, 2, 0)), (g, 0, SegmentKey(0, 1, 0, 2, 1))], gs)
dequant_accumulate([(g0c, g0m), (g1c, g1m)], n, gs, 2)                     # K4, 2 sources
xi = torch.randn(n, device=dev) * 0.02
dequant_accumulate_lattice([(g0c, g0m)], n, gs, 1, xi, LatticeStep(0.25, 1e-4, shift_key(0, 1, 0)))  # K4 + lattice
torch.cuda.synchronize()
print("prof_rows: done")
