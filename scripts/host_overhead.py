"""Host-side cost of one group collective call (a GPT-block-shaped group: 4 dense weights +
8 full-precision pieces; under torchrun each rank holds 1/world of it): microseconds of host time per C-ABI call, per
comm.*_pieces wrapper call, and per CUDA launch (torch empty-kernel baseline)."""
import ctypes
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_02390_b200 import _lib  # noqa: E402
from paper_2302_02390_b200.comm import QSDPComm  # noqa: E402
from paper_2302_02390_b200.quantize import QuantSpec, SegmentKey  # noqa: E402

d = int(os.environ.get("D", "2048"))
world = int(os.environ.get("WORLD_SIZE", "1"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
if world > 1:
    import torch.distributed as dist
    dist.init_process_group("nccl", device_id=dev)
    d = d // world  # per-rank shard of the block's parameters
dense = [3 * d * d, d * d, 4 * d * d, 4 * d * d]
raw = [d, d, 3 * d, d, d, d, 4 * d, d]
offs, off = [], 0
for n in dense + raw:
    offs.append(off)
    off += n
stride = off
comm = QSDPComm(sum(dense) + 4 * 1040 + 4 * (sum(raw) + 64), QuantSpec(8, 1024, "shift"),
                QuantSpec(8, 1024, "uniform_stochastic"), device=dev)
srcs = [torch.randn(n, device=dev) for n in dense + raw]
out = torch.empty(world * stride, dtype=torch.bfloat16, device=dev)
rs_out = torch.empty(stride, dtype=torch.float32, device=dev)
pieces = (_lib.Piece * len(srcs))()
for k, (x, o) in enumerate(zip(srcs, offs)):
    pieces[k] = _lib.Piece(x.data_ptr(), o, x.numel(), 0 if k < len(dense) else 1, 0)
grad = torch.randn(world * stride, device=dev)  # rank-major gradient for the reduce-scatter
rs_pieces = (_lib.Piece * len(srcs))()
for k, o in enumerate(offs):
    rs_pieces[k] = _lib.Piece(grad.data_ptr() + 4 * o, o, srcs[k].numel(), 0 if k < len(dense) else 1, 0)
key = _lib.Key(0, 0, 1, 0, 0)
kp = ctypes.byref(key)
L = _lib.lib()
s = torch.cuda.current_stream().cuda_stream


def bench(fn, n=200):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return (t1 - t0) / n * 1e6


res = {
    "capi_all_gather_pieces_us": bench(lambda: _lib.check(L.qsdp_all_gather_pieces(
        comm._h, pieces, len(srcs), _lib.F32, stride, kp, out.data_ptr(), 2, s))),
    "capi_reduce_scatter_pieces_us": bench(lambda: _lib.check(L.qsdp_reduce_scatter_pieces(
        comm._h, rs_pieces, len(srcs), _lib.F32, stride, kp, rs_out.data_ptr(), 0, s))),
    "wrapper_all_gather_pieces_us": bench(lambda: comm.all_gather_pieces(
        [(x, o, x.numel(), k >= len(dense)) for k, (x, o) in enumerate(zip(srcs, offs))], stride,
        SegmentKey(0, 0, 1, 0, 0), out)),
    "torch_empty_kernel_launch_us": bench(lambda: torch.cuda._sleep(0)),
}
if int(os.environ.get("RANK", "0")) == 0:
    print({"world": world, **{k: round(v, 2) for k, v in res.items()}})
if world > 1:
    dist.barrier()
    dist.destroy_process_group()
