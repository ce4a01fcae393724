"""Per-kernel device times of the QSDP collectives at world W (torch profiler /
CUPTI; no ncu on multi-rank runs).  Rank 0 prints the kernel table.

    python -m torch.distributed.run --nproc-per-node W --master-addr 127.0.0.1 scripts/comm_kernel_times.py
"""
import collections
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_02390_b200.comm import QSDPComm, plan_segments  # noqa: E402
from paper_2302_02390_b200.gpt import dense_groups  # noqa: E402
from paper_2302_02390_b200.quantize import QuantSpec, SegmentKey  # noqa: E402


def main():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    wspec, gspec = QuantSpec(8, 1024, "shift"), QuantSpec(8, 1024, "uniform_stochastic")
    groups = dense_groups("gpt2-125m")
    state, max_seg = [], 0
    for g in groups:
        segs = plan_segments(g.numel, world, 1024)
        max_seg = max(max_seg, max(n for _, n in segs))
        s, n = segs[rank]
        state.append(dict(segs=segs, n=n, shard=torch.randn(max(n, 1), device=dev)[:n] * 0.02,
                          grad=torch.randn(g.numel, device=dev) * 1e-3, full=torch.empty(g.numel, device=dev),
                          gshard=torch.empty(max(n, 1), device=dev)))
    comm = QSDPComm(max_seg, wspec, gspec, device=dev)

    mode = os.environ.get("MODE", "both")

    def step(t):
        if mode in ("both", "ag"):
            for gi, st in enumerate(state):
                comm.all_gather(st["shard"], st["segs"], SegmentKey(0, t, gi, 0, 0), st["full"])
        if mode in ("both", "rs"):
            for gi, st in enumerate(state):
                comm.reduce_scatter(st["grad"], st["segs"], SegmentKey(0, t, gi, 2, rank), st["gshard"])

    for t in range(3):
        step(t)
    torch.cuda.synchronize()
    reps = 5
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for t in range(reps):
            step(10 + t)
        torch.cuda.synchronize()
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            name = e.name.split("<")[0].split("(")[0].replace("void ", "").replace("qsdp::", "")
            tot[name] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
            cnt[name] += 1
    if rank == 0:
        print(f"world {world} mode {mode}: per step, us")
        for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
            print(f"  {k:40s} {v / reps:9.1f} us  ({cnt[k] // reps} launches)")
    comm.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
