"""Step throughput of the hierarchical communicator on the
bench workload (GPT-2 125M, 13 groups, AG fwd + AG bwd + RS per step), eager,
CUDA events, max over ranks.  On one box the "inter-node" level runs over
NVLink too, so this measures the protocol's cost, not an IB fabric.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 scripts/hier_bench.py [node_size]
"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_02390_b200.comm import plan_segments  # noqa: E402
from paper_2302_02390_b200.comm_hier import HierComm  # noqa: E402
from paper_2302_02390_b200.gpt import dense_groups  # noqa: E402
from paper_2302_02390_b200.quantize import QuantSpec, SegmentKey  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, world = dist.get_rank(), dist.get_world_size()
    node_size = int(sys.argv[1]) if len(sys.argv) > 1 else world
    groups = dense_groups("gpt2-125m")
    state, max_seg = [], 0
    for g in groups:
        segs = plan_segments(g.numel, world, 1024)
        max_seg = max(max_seg, max(n for _, n in segs))
        s, n = segs[rank]
        state.append(dict(segs=segs, shard=torch.randn(max(n, 1), device=dev)[:n] * 0.02,
                          grad=torch.randn(g.numel, device=dev) * 1e-3, full=torch.empty(g.numel, device=dev),
                          gshard=torch.empty(max(n, 1), device=dev)))
    comm = HierComm(max_seg, QuantSpec(8, 1024, "shift"), QuantSpec(8, 1024, "uniform_stochastic"), node_size, dev)
    flush = torch.empty(64 << 20, dtype=torch.int32, device=dev)

    def step(t):
        for gi, st in enumerate(state):
            comm.all_gather(st["shard"], st["segs"], SegmentKey(0, t, gi, 0, 0), st["full"])
        for gi in range(len(state) - 1, -1, -1):
            st = state[gi]
            comm.all_gather(st["shard"], st["segs"], SegmentKey(0, t, gi, 1, 0), st["full"])
            comm.reduce_scatter(st["grad"], st["segs"], SegmentKey(0, t, gi, 2, rank), st["gshard"])

    for t in range(3):
        step(t)
    torch.cuda.synchronize()
    tot, reps = 0.0, 10
    for t in range(reps):
        flush.fill_(t)
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        step(100 + t)
        b.record()
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    ms = torch.tensor([tot / reps], device=dev, dtype=torch.float64)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    N = sum(g.numel for g in groups)
    if rank == 0:
        print(json.dumps({"world": world, "node_size": node_size, "ms_per_step": round(float(ms.item()), 4),
                          "value_gbs": round(world * 12.0 * N / (float(ms.item()) * 1e-3) / 1e9, 1)}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
