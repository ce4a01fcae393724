"""Run each hot-path kernel on a GPT-2-small-sized bucket set (for ncu / timing).

    python scripts/prof_kernels.py [--n ELEMS] [--reps R]
Launch order per rep: K1 (shift quantize), K3 (dequantize), K2 (stochastic
quantize), K4 (dequant-accumulate, P=1).  Prints CUDA-event GB/s per kernel.
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_02390_b200.quantize import (QuantSpec, SegmentKey, codes_bytes, dequant_accumulate,  # noqa: E402
                                            dequantize_segments, num_buckets, quantize_segments)

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=38633472)  # wte + wpe of GPT-2 small
ap.add_argument("--reps", type=int, default=11)
ap.add_argument("--bits", type=int, default=8)
ap.add_argument("--gbits", type=int, default=8)
ap.add_argument("--bucket", type=int, default=1024)
ap.add_argument("--levels", action="store_true", help="also time the levels-mode kernels (LQ/LD) and learn_levels")
a = ap.parse_args()
dev = torch.device("cuda", 0)
n = a.n
x = torch.randn(n, device=dev) * 0.02
g = torch.randn(n, device=dev) * 1e-3
out = torch.empty(n, device=dev)
ws, gs = QuantSpec(a.bits, a.bucket, "shift"), QuantSpec(a.gbits, a.bucket, "uniform_stochastic")
wq = (torch.empty(codes_bytes(n, ws) + 16, dtype=torch.uint8, device=dev),
      torch.empty((num_buckets(n, a.bucket), 3), device=dev))
gq = (torch.empty(codes_bytes(n, gs) + 16, dtype=torch.uint8, device=dev),
      torch.empty((num_buckets(n, a.bucket), 3), device=dev))
cbw = codes_bytes(n, ws) + 12 * num_buckets(n, a.bucket)
cbg = codes_bytes(n, gs) + 12 * num_buckets(n, a.bucket)
kern = {
    "K1": (lambda s: quantize_segments([(x, 0, SegmentKey(0, s, 0, 0, 0))], ws, out=[wq]), 4 * n + cbw),
    "K3": (lambda s: dequantize_segments([(wq[0], wq[1], n, out)], ws), cbw + 4 * n),
    "K2": (lambda s: quantize_segments([(g, 0, SegmentKey(0, s, 0, 2, 0))], gs, out=[gq]), 4 * n + cbg),
    "K4": (lambda s: dequant_accumulate([gq], n, gs, 1, out=out), cbg + 4 * n),
}
if a.levels:
    from paper_2302_02390_b200.levels import LevelTable, dequantize_levels, learn_levels, quantize_levels_segments
    ls = QuantSpec(a.bits, a.bucket, "levels")
    u = torch.rand(200000, device=dev, dtype=torch.float64)
    table = learn_levels(u, LevelTable.uniform(a.bits))
    lq = (torch.empty(codes_bytes(n, ls) + 16, dtype=torch.uint8, device=dev),
          torch.empty((num_buckets(n, a.bucket), 3), device=dev))
    cbl = codes_bytes(n, ls) + 12 * num_buckets(n, a.bucket)
    kern["LQ"] = (lambda s: quantize_levels_segments([x], ls, table, out=[lq]), 4 * n + cbl)
    kern["LD"] = (lambda s: dequantize_levels(lq[0], lq[1], n, ls, table, dtype=torch.float32, out=out), cbl + 4 * n)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    learn_levels(u, LevelTable.uniform(a.bits))
    e1.record()
    torch.cuda.synchronize()
    print(f"learn_levels: {u.numel()} values, {a.bits}-bit table: {e0.elapsed_time(e1):.2f} ms "
          f"({u.numel() / e0.elapsed_time(e1) / 1e3:.2f} M values/s)")
res = {k: 0.0 for k in kern}
for r in range(a.reps):
    for k, (fn, nb) in kern.items():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(2_000_000)  # GPU busy while the host enqueues: the events time the kernel, not the launch
        e0.record()
        fn(r)
        e1.record()
        torch.cuda.synchronize()
        if r > 0:
            res[k] += e0.elapsed_time(e1)
for k, (fn, nb) in kern.items():
    t = res[k] / max(1, a.reps - 1)
    print(f"{k}: {t:.4f} ms  {nb / t / 1e6:.1f} GB/s")
