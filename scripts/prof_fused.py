"""World-1 collectives as the bench step runs them (one fused quantizer launch each), for ncu.

    python scripts/prof_fused.py [--n ELEMS] [--reps R]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_02390_b200.comm import QSDPComm  # noqa: E402
from paper_2302_02390_b200.quantize import QuantSpec, SegmentKey  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=38633472)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
dev = torch.device("cuda", 0)
n = a.n
x = torch.randn(n, device=dev) * 0.02
g = torch.randn(n, device=dev) * 1e-3
full = torch.empty(n, device=dev)
shard = torch.empty(n, device=dev)
comm = QSDPComm(n, QuantSpec(8, 1024, "shift"), QuantSpec(8, 1024, "uniform_stochastic"), device=dev)
for r in range(a.reps):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    torch.cuda._sleep(4_000_000)  # GPU busy while the host enqueues: the events time the kernels, not the launches
    ev[0].record()
    comm.all_gather(x, [(0, n)], SegmentKey(0, r, 0, 0, 0), full)
    ev[1].record()
    comm.reduce_scatter(g, [(0, n)], SegmentKey(0, r, 0, 2, 0), shard)
    ev[2].record()
    torch.cuda.synchronize()
    print(f"AG {ev[0].elapsed_time(ev[1]) * 1e3:.1f} us ({8 * n / ev[0].elapsed_time(ev[1]) / 1e6:.0f} GB/s)  "
          f"RS {ev[1].elapsed_time(ev[2]) * 1e3:.1f} us ({8 * n / ev[1].elapsed_time(ev[2]) / 1e6:.0f} GB/s)")
comm.close()
