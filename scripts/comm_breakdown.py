"""Where a QSDP step's time goes at world W: graphs of only the all-gathers,
only the reduce-scatters, and tiny collectives (barrier + launch cost).

    python -m torch.distributed.run --nproc-per-node W --master-addr 127.0.0.1 scripts/comm_breakdown.py
"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_02390_b200.comm import QSDPComm, plan_segments  # noqa: E402
from paper_2302_02390_b200.gpt import dense_groups  # noqa: E402
from paper_2302_02390_b200.quantize import QuantSpec, SegmentKey, advance_counter  # noqa: E402


def main():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    wspec, gspec = QuantSpec(8, 1024, "shift"), QuantSpec(8, 1024, "uniform_stochastic")
    groups = dense_groups(os.environ.get("MODEL", "gpt2-125m"))
    state, max_seg = [], 0
    for g in groups:
        segs = plan_segments(g.numel, world, 1024)
        max_seg = max(max_seg, max(n for _, n in segs))
        s, n = segs[rank]
        state.append(dict(segs=segs, n=n, shard=torch.randn(max(n, 1), device=dev)[:n] * 0.02,
                          grad=torch.randn(g.numel, device=dev) * 1e-3, full=torch.empty(g.numel, device=dev),
                          gshard=torch.empty(max(n, 1), device=dev)))
    tiny = plan_segments(1024 * world, world, 1024)
    tin, tout = torch.randn(1024, device=dev), torch.empty(1024 * world, device=dev)
    ctr = torch.zeros(1, dtype=torch.int64, device=dev)
    comm = QSDPComm(max_seg, wspec, gspec, device=dev)
    comm.set_step_source(ctr)
    flush = torch.empty(64 << 20, dtype=torch.int32, device=dev)

    def ag():
        for gi, st in enumerate(state):
            comm.all_gather(st["shard"], st["segs"], SegmentKey(0, 0, gi, 0, 0), st["full"])
        advance_counter(ctr)

    def rs():
        for gi, st in enumerate(state):
            comm.reduce_scatter(st["grad"], st["segs"], SegmentKey(0, 0, gi, 2, rank), st["gshard"])
        advance_counter(ctr)

    def tiny_ag():
        for gi in range(len(state)):
            comm.all_gather(tin, tiny, SegmentKey(0, 0, gi, 0, 0), tout)
        advance_counter(ctr)

    res = {"world": world, "groups": len(state)}
    for name, fn in (("allgather_x13", ag), ("reducescatter_x13", rs), ("tiny_allgather_x13", tiny_ag)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        g.replay()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        tot = 0.0
        for r in range(20):
            flush.fill_(r)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            torch.cuda.synchronize()
            tot += a.elapsed_time(b)
        t = torch.tensor([tot / 20], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res[name + "_ms"] = round(float(t.item()), 4)
    if rank == 0:
        print(json.dumps(res), flush=True)
    comm.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
