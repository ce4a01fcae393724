"""Hierarchical C1/C2 under torchrun: every rank checks its
all-gather output and its reduce-scatter shard bit-exactly against the
oracle's protocol, for each node shape that divides the world size.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tests/dist_hier_check.py
"""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import oracle as O  # noqa: E402  (checker only)
from paper_2302_02390_b200.comm import plan_segments  # noqa: E402
from paper_2302_02390_b200.comm_hier import HierComm  # noqa: E402
from paper_2302_02390_b200.quantize import QuantSpec, SegmentKey  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, world = dist.get_rank(), dist.get_world_size()
    fails = 0
    for node_size in [d for d in (1, 2, 4, 8) if world % d == 0 and d <= world]:
        for size, bucket, wb, gb, pad in [(1 << 20, 1024, 8, 8, 1024), (300007, 256, 4, 4, 1), (77777, 100, 6, 5, 1)]:
            segs = plan_segments(size, world, pad)
            comm = HierComm(max(n for _, n in segs), QuantSpec(wb, bucket, "shift"),
                            QuantSpec(gb, bucket, "uniform_stochastic"), node_size, device=dev)
            full = (np.random.default_rng(size).standard_normal(size) * 0.02).astype(np.float32)
            grads = [(np.random.default_rng(size + 1 + p).standard_normal(size) * 1e-3).astype(np.float32)
                     for p in range(world)]
            s, n = segs[rank]
            for step in range(2):
                out = torch.empty(size, dtype=torch.float32, device=dev)
                comm.all_gather(torch.from_numpy(full[s:s + n]).to(dev), segs, SegmentKey(3, step, 1, 0, 0), out)
                exp = np.zeros(size)
                for sq, nq in segs:
                    if nq:
                        c, m, _ = O.quantize_segment(full[sq:sq + nq], sq, bucket, wb, 0, (3, step, 1, 0, 0), 8)
                        exp[sq:sq + nq] = O.dequantize_segment(c, m, nq, bucket, wb, 8)
                ok_ag = np.array_equal(out.cpu().numpy(), exp.astype(np.float32))
                sh = torch.empty(max(n, 1), dtype=torch.float32, device=dev)
                comm.reduce_scatter(torch.from_numpy(grads[rank]).to(dev), segs, SegmentKey(3, step, 1, 2, rank), sh)
                acc = np.zeros(n)
                for p in range(world):
                    if n:
                        c, m, _ = O.quantize_segment(grads[p][s:s + n], s, bucket, gb, 1, (3, step, 1, 2, p), 8)
                        acc = acc + O.dequantize_segment(c, m, n, bucket, gb, 8)
                ok_rs = np.array_equal(sh[:n].cpu().numpy(), (acc / world).astype(np.float32))
                if not (ok_ag and ok_rs):
                    fails += 1
                    print(f"rank {rank} node_size {node_size} size {size} step {step}: ag {ok_ag} rs {ok_rs}", flush=True)
    t = torch.tensor([fails], device=dev)
    dist.all_reduce(t)
    if rank == 0:
        print(f"dist_hier_check world={world}: {'OK' if t.item() == 0 else 'FAILED'}", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if t.item() == 0 else 1)


if __name__ == "__main__":
    main()
