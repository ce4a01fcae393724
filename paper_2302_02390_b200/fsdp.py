"""QSDP inside PyTorch FSDP2: custom all-gather / reduce-scatter comms (H1).

Replaces the reference's per-layer hook call order (``forward_layer`` /
``backward_layer``, pkg/src/qsdp/sharded.py:437-469; Alg. 3 of the paper)
with FSDP2's own scheduling: every ``fully_shard``-ed module group gets a
:class:`QSDPAllGather` and a :class:`QSDPReduceScatter`
(``FSDPModule.set_custom_all_gather`` / ``set_custom_reduce_scatter``,
torch/distributed/fsdp/_fully_shard/_fully_shard.py:458-482).  FSDP2 runs
them on its dedicated all-gather and reduce-scatter streams, prefetching the
next group's gather while the current group computes, so the quantized
collectives overlap compute as in the paper.

Keys follow the reference protocol: weights (root, step, group, phase, worker 0,
start) with phase 0 in forward and 1 in the backward re-gather; gradients
(root, step, group, PHASE_GRAD, rank, start).  The step is the host-side
training step (:meth:`QSDPContext.next_step`).

FSDP2 flattens each group's parameters into one per-rank buffer (padded to
equal shards), so the quantized buckets run over that flat buffer.
"""

from __future__ import annotations

import torch
import torch.distributed as dist
from torch.distributed.fsdp._fully_shard._fsdp_api import AllGather, ReduceScatter

from .comm import QSDPComm, record_allgather, record_reducescatter
from .quantize import QuantSpec, SegmentKey
from .sharded import PHASE_GRAD, PHASE_W_BWD, PHASE_W_FWD, CommLedger, LedgerEntry

__all__ = ["QSDPContext", "QSDPAllGather", "QSDPReduceScatter", "apply_qsdp"]


class QSDPContext:
    """Shared state of one QSDP training run: communicators, step and phase."""

    def __init__(self, max_shard_numel: int, wspec: QuantSpec, gspec: QuantSpec, root_seed: int = 0,
                 group: dist.ProcessGroup | None = None, device: torch.device | None = None,
                 weight_levels=None, sm_budget: int | None = None):
        self.wspec, self.gspec = wspec, gspec
        self.root_seed = root_seed
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        # FSDP2 issues all-gathers and reduce-scatters on different streams: one
        # communicator (slots + device epoch) per stream keeps each sequence ordered.
        # wspec.inner == "levels": the all-gather codes weights through a learned
        # table (levels.LevelTable, e.g. levels.learn_weight_levels(model weights))
        self.ag = QSDPComm(max_shard_numel, wspec, gspec, group=group, device=device, weight_levels=weight_levels)
        self.rs = QSDPComm(max_shard_numel, wspec, gspec, group=group, device=device)
        # the comm streams overlap backward / forward compute: cap their SMs
        if sm_budget is None:
            import os
            sm_budget = int(os.environ.get("QSDP_SM_BUDGET", "0"))
        self.ag.set_sm_budget(sm_budget)
        self.rs.set_sm_budget(sm_budget)
        self.step = 0
        self.phase = PHASE_W_FWD
        self.calls = {"allgather": 0, "reducescatter": 0}
        # the reference's per-step communication ledger (sharded.py:115-181)
        self.ledger = CommLedger()
        self.entry = LedgerEntry(step=0)

    def forward(self):
        self.phase = PHASE_W_FWD

    def backward(self):
        self.phase = PHASE_W_BWD

    def next_step(self, step_time_s: float = 0.0):
        self.entry.step_time_s = step_time_s
        self.ledger.append(self.entry)
        self.step += 1
        self.entry = LedgerEntry(step=self.step)
        self.phase = PHASE_W_FWD

    def close(self):
        self.ag.close()
        self.rs.close()


class QSDPAllGather(AllGather):
    """Quantized all-gather of one FSDP2 group (C1)."""

    def __init__(self, ctx: QSDPContext, layer: int):
        self.ctx, self.layer = ctx, layer

    def allocate(self, size, *, dtype, device):
        return torch.empty(*size, dtype=dtype, device=device)

    def __call__(self, output_tensor, input_tensor, group, async_op=False):
        if input_tensor.dtype not in (torch.float32,):
            raise ValueError("QSDP all-gather expects fp32 sharded parameters (param_dtype=None)")
        world = group.size()
        n = input_tensor.numel()
        segs = [(p * n, n) for p in range(world)]
        c = self.ctx
        c.ag.all_gather(input_tensor, segs, SegmentKey(c.root_seed, c.step, self.layer, c.phase, 0), output_tensor)
        c.calls["allgather"] += 1
        record_allgather(c.entry, f"group{self.layer}", segs, c.wspec)
        return None


class QSDPReduceScatter(ReduceScatter):
    """Quantized reduce-scatter of one FSDP2 group's gradients (C2): average of the
    dequantized contributions of every rank (sharded.py:375-433)."""

    def __init__(self, ctx: QSDPContext, layer: int):
        self.ctx, self.layer = ctx, layer

    def allocate(self, size, *, dtype, device):
        return torch.empty(*size, dtype=dtype, device=device)

    def __call__(self, output_tensor, input_tensor, group, op, async_op=False):
        if op not in (dist.ReduceOp.AVG,) and getattr(op, "op", op) != dist.ReduceOp.AVG:
            raise ValueError("QSDP reduce-scatter computes the average (ReduceOp.AVG)")
        if input_tensor.dtype != torch.float32:
            raise ValueError("QSDP reduce-scatter expects fp32 gradients (reduce_dtype=float32)")
        world = group.size()
        n = output_tensor.numel()
        segs = [(p * n, n) for p in range(world)]
        c = self.ctx
        c.rs.reduce_scatter(input_tensor, segs, SegmentKey(c.root_seed, c.step, self.layer, PHASE_GRAD, c.rank),
                            output_tensor)
        c.calls["reducescatter"] += 1
        record_reducescatter(c.entry, f"group{self.layer}", segs, c.gspec)
        return None


def apply_qsdp(modules, ctx: QSDPContext) -> None:
    """Install QSDP comms on ``fully_shard``-ed modules (index = key ``layer``)."""
    for i, m in enumerate(modules):
        m.set_custom_all_gather(QSDPAllGather(ctx, i))
        m.set_custom_reduce_scatter(QSDPReduceScatter(ctx, i))
