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

**Per-parameter protocol.**  FSDP2 flattens a group's parameters into one
per-rank buffer: parameter k's dim-0-padded shard at a fixed offset, the same on
every rank (``foreach_all_gather`` / ``foreach_reduce_scatter_copy_in``,
torch/distributed/fsdp/_fully_shard/_fsdp_collectives.py:237-290, 667-675).
The comms walk that layout (:func:`group_layout`) and treat each parameter as
the reference treats a layer:

* dense weights (2-D: linear / embedding matrices) are quantized -- weights with
  the random-shift quantizer, gradients with the stochastic one -- keyed
  (root, step, group, phase, worker, start) with ``start`` = the parameter
  piece's offset in the gathered buffer (sharded.py:323-358, 386-413);
* biases and norm parameters (1-D) travel at full precision (sharded.py:359-371,
  414-429) inside the same group collective (``qsdp_piece.raw``): the all-gather
  casts each rank's fp32 master piece to the parameter dtype (RNE, the cast FSDP2's
  copy-in does, so these are bit-identical to the unquantized path), the
  reduce-scatter averages the ranks' contributions in rank order in fp64 and rounds
  once (the reference's ``acc + vals ... / P``).  One C call, one barrier per
  group: no separate NCCL collective and no host-side gather/scatter of the pieces.

With ``param_dtype=bf16`` (bf16 compute, the FSDP2 mixed-precision baseline) the
all-gather quantizes the fp32 master shard (``FSDPParam._sharded_param_data``,
not FSDP2's bf16 copy-in) and writes the dequantized weights as bf16
(RNE of the fp32 value == float32(reference fp64)); gradients are reduced in fp32
(``reduce_dtype``).  Keys use the host step and the forward / backward phase.
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass

import torch
import torch.distributed as dist
from torch.distributed.fsdp._fully_shard._fsdp_api import AllGather, ReduceScatter

from .comm import QSDPComm, record_allgather, record_reducescatter
from .quantize import QuantSpec, SegmentKey
from .sharded import PHASE_GRAD, PHASE_W_BWD, PHASE_W_FWD, CommLedger, LedgerEntry, Transfer

__all__ = ["QSDPContext", "QSDPAllGather", "QSDPReduceScatter", "apply_qsdp", "group_layout", "ParamSlot"]


@dataclass
class ParamSlot:
    """One parameter of a FSDP2 group in the per-rank flat buffer."""

    name: str
    offset: int      # element offset within a rank's flat shard
    numel: int       # padded shard numel (identical on every rank)
    dense: bool      # quantized (2-D weight) or full precision (bias / norm)
    fsdp_param: object


def group_layout(module) -> list[ParamSlot]:
    """The flat layout FSDP2 all-gathers / reduce-scatters for ``module``'s group:
    parameters in ``fsdp_params`` order, each its padded sharded numel."""
    state = module._get_fsdp_state()
    pg = state._fsdp_param_group
    if pg is None:
        return []
    slots, off = [], 0
    for fp in pg.fsdp_params:
        n = fp.padded_sharded_param_size.numel()
        name = getattr(getattr(fp, "_module_info", None), "param_name", "param")
        slots.append(ParamSlot(name, off, n, len(fp._orig_size) >= 2, fp))
        off += n
    return slots


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
            sm_budget = int(os.environ.get("QSDP_SM_BUDGET", "0"))
        self.ag.set_sm_budget(sm_budget)
        self.rs.set_sm_budget(sm_budget)
        ag_ctas = int(os.environ.get("QSDP_AG_CTAS", "0"))  # all-gather quantizer CTAs per SM (0 = occupancy)
        if ag_ctas:
            self.ag.set_ctas_per_sm(ag_ctas)
        self.step = 0
        self.phase = PHASE_W_FWD
        self.calls = {"allgather": 0, "reducescatter": 0}
        # host time inside the comm hooks (and inside their C-ABI calls)
        self.host_s = {"allgather": 0.0, "reducescatter": 0.0, "allgather_capi": 0.0, "reducescatter_capi": 0.0}
        self.capi_samples: list[float] = []  # per-call host time of the all-gather C-ABI call
        self.layouts: dict[int, list[ParamSlot]] = {}
        self.param_bits = None  # width of the full-precision all-gather (set from the param dtype)
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

    def record(self, template: LedgerEntry) -> None:
        """Add one collective's (cached) ledger records to the current step's entry."""
        e = self.entry
        e.transfers.extend(template.transfers)
        e.allgather_bits += template.allgather_bits
        e.reducescatter_bits += template.reducescatter_bits
        e.allgather_payload_bits += template.allgather_payload_bits
        e.reducescatter_payload_bits += template.reducescatter_payload_bits
        e.allgather_events += 1 if template.allgather_events else 0
        e.reducescatter_events += 1 if template.reducescatter_events else 0

    def close(self):
        self.ag.close()
        self.rs.close()


class _LayerPlan:
    """Per-(group, world) host state built on the first collective and reused: the C-ABI
    piece array (quantized and full-precision pieces) and the ledger records (FSDP2 drives
    these comms from its Python hooks, so per-call host work is on the step's critical
    path -- the 1.3B step is host-bound)."""

    def __init__(self, ctx: "QSDPContext", layer: int, world: int, stride: int, device, kind: str):
        import ctypes
        from . import _lib
        slots = ctx.layouts[layer]
        if sum(s.numel for s in slots) != stride:
            raise ValueError("FSDP2 collective buffer does not match the group's parameter layout")
        self.slots = [s for s in slots if s.numel]
        self.pieces = (_lib.Piece * max(1, len(self.slots)))()
        for k, s in enumerate(self.slots):
            self.pieces[k] = _lib.Piece(None, s.offset, s.numel, 0 if s.dense else 1, 0)
        self.n = len(self.slots)
        self.masters = ()
        self.base = None
        self.key = _lib.Key(ctx.root_seed, 0, layer, 0, 0)
        self.keyp = ctypes.byref(self.key)
        # the reference's ledger records of this collective (sharded.py:349-371, 403-429)
        probe = LedgerEntry(step=0)
        for s in self.slots:
            if not s.dense:
                continue
            if kind == "allgather":
                record_allgather(probe, f"group{layer}.{s.name}", [(0, s.numel)] * world, ctx.wspec)
            else:
                record_reducescatter(probe, f"group{layer}.{s.name}", [(0, s.numel)] * world, ctx.gspec)
        for s in slots:
            if s.dense or not s.numel:
                continue
            if kind == "allgather":
                width = 32 if ctx.param_bits is None else ctx.param_bits
                for _ in range(world):
                    probe.record(Transfer("allgather", f"group{layer}.{s.name}", width, s.numel * width // 8,
                                          world - 1, s.numel * width))
            else:
                for _ in range(world - 1):
                    probe.record(Transfer("reducescatter", f"group{layer}.{s.name}", 32, s.numel * 4, 1, s.numel * 32))
        self.ledger = probe


class QSDPAllGather(AllGather):
    """Quantized all-gather of one FSDP2 group (C1): the group's dense weights in one
    group collective (qsdp_all_gather_pieces), biases / norms gathered at full precision."""

    def __init__(self, ctx: QSDPContext, layer: int):
        self.ctx, self.layer = ctx, layer
        self.plans = {}

    def allocate(self, size, *, dtype, device):
        return torch.empty(*size, dtype=dtype, device=device)

    def __call__(self, output_tensor, input_tensor, group, async_op=False):
        from . import _lib
        from .quantize import _DTYPE_CODE
        t0 = time.perf_counter()
        c = self.ctx
        if output_tensor.dtype not in (torch.float32, torch.bfloat16):
            raise ValueError("QSDP all-gather writes fp32 or bf16 parameters")
        world = group.size()
        n_in = input_tensor.numel()
        pl = self.plans.get((world, n_in))
        if pl is None:
            pl = self.plans[(world, n_in)] = _LayerPlan(c, self.layer, world, n_in, output_tensor.device, "allgather")
        masters = [s.fsdp_param._sharded_param_data for s in pl.slots]  # fp32 master shards
        ptrs = tuple(m.data_ptr() for m in masters)
        if ptrs != pl.masters:
            for k, m in enumerate(masters):
                if m.dtype != torch.float32 or m.numel() != pl.slots[k].numel:
                    raise ValueError("QSDP all-gather expects fp32 sharded parameters")
                pl.pieces[k].src = ptrs[k]
            pl.masters = ptrs
        if not pl.n:
            pass
        elif c.wspec.inner != "levels":  # the whole group: one quantize, one barrier, one dequant
            pl.key.step, pl.key.phase = c.step, c.phase
            stream, optr, odt = torch.cuda.current_stream().cuda_stream, output_tensor.data_ptr(), _DTYPE_CODE[output_tensor.dtype]
            t1 = time.perf_counter()
            rc = _lib.hot().qsdp_all_gather_pieces(c.ag._h, pl.pieces, pl.n, _lib.F32, n_in, pl.keyp, optr, odt, stream)
            dt = time.perf_counter() - t1
            c.host_s["allgather_capi"] += dt
            if len(c.capi_samples) < 4096:
                c.capi_samples.append(dt)
            _lib.check(rc)
        else:  # learned levels: one collective per weight, full-precision pieces in one more
            key = SegmentKey(c.root_seed, c.step, self.layer, c.phase, 0)
            raw = [(m, s.offset, s.numel, True) for m, s in zip(masters, pl.slots) if not s.dense]
            for m, s in zip(masters, pl.slots):
                if s.dense:
                    c.ag.all_gather(m, [(q * n_in + s.offset, s.numel) for q in range(world)], key,
                                    output_tensor[s.offset:])
            if raw:
                c.ag.all_gather_pieces(raw, n_in, key, output_tensor)
        c.record(pl.ledger)
        c.calls["allgather"] += 1
        c.host_s["allgather"] += time.perf_counter() - t0
        return None


class QSDPReduceScatter(ReduceScatter):
    """Quantized reduce-scatter of one FSDP2 group's gradients (C2): the average of the
    dequantized contributions of every rank (sharded.py:375-433) for the group's dense
    weights in one group collective; biases / norms reduced at full precision."""

    def __init__(self, ctx: QSDPContext, layer: int):
        self.ctx, self.layer = ctx, layer
        self.plans = {}

    def allocate(self, size, *, dtype, device):
        return torch.empty(*size, dtype=dtype, device=device)

    def __call__(self, output_tensor, input_tensor, group, op, async_op=False):
        from . import _lib
        t0 = time.perf_counter()
        if op not in (dist.ReduceOp.AVG,) and getattr(op, "op", op) != dist.ReduceOp.AVG:
            raise ValueError("QSDP reduce-scatter computes the average (ReduceOp.AVG)")
        if input_tensor.dtype != torch.float32 or output_tensor.dtype != torch.float32:
            raise ValueError("QSDP reduce-scatter expects fp32 gradients (reduce_dtype=float32)")
        c = self.ctx
        world = group.size()
        n_out = output_tensor.numel()
        pl = self.plans.get((world, n_out))
        if pl is None:
            pl = self.plans[(world, n_out)] = _LayerPlan(c, self.layer, world, n_out, output_tensor.device,
                                                         "reducescatter")
        base = input_tensor.data_ptr()
        if base != pl.base:
            for k, s in enumerate(pl.slots):
                pl.pieces[k].src = base + 4 * s.offset
            pl.base = base
        pl.key.step, pl.key.phase, pl.key.worker = c.step, PHASE_GRAD, c.rank
        if pl.n:
            stream, optr = torch.cuda.current_stream().cuda_stream, output_tensor.data_ptr()
            t1 = time.perf_counter()
            rc = _lib.hot().qsdp_reduce_scatter_pieces(c.rs._h, pl.pieces, pl.n, _lib.F32, n_out, pl.keyp, optr,
                                                       _lib.F32, stream)
            c.host_s["reducescatter_capi"] += time.perf_counter() - t1
            _lib.check(rc)
        c.record(pl.ledger)
        c.calls["reducescatter"] += 1
        c.host_s["reducescatter"] += time.perf_counter() - t0
        return None


def apply_qsdp(modules, ctx: QSDPContext, param_dtype=None) -> None:
    """Install QSDP comms on ``fully_shard``-ed modules (index = key ``layer``)."""
    ctx.param_bits = None if param_dtype is None else torch.finfo(param_dtype).bits
    for i, m in enumerate(modules):
        ctx.layouts[i] = group_layout(m)
        m.set_custom_all_gather(QSDPAllGather(ctx, i))
        m.set_custom_reduce_scatter(QSDPReduceScatter(ctx, i))
