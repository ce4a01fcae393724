"""GPT training step on FSDP2, with QSDP quantized collectives or the
unquantized FSDP2 baseline (BASELINE.json configs: GPT-2 small / medium /
1.3B on synthetic tokens).

Random-init GPT-2 architecture (transformers ``GPT2LMHeadModel``; there is no
network for checkpoints), synthetic tokens uniform over the vocabulary, fp32
master parameters sharded by FSDP2 with bf16 autocast compute, AdamW
(lr 6e-4, betas 0.9/0.95 -- the paper's 125M settings).
Both modes use the identical setup; only the all-gather / reduce-scatter
comms differ (fp32 NCCL vs QSDP w8/g8 over NVLink peer memory).
"""

from __future__ import annotations

import math

import torch
import torch.distributed as dist

from .gpt import GPT_CONFIGS
from .quantize import QuantSpec

__all__ = ["build_model", "shard_model", "run_training"]


def build_model(model: str, device: torch.device, seed: int = 0, layers: int | None = None):
    from transformers import GPT2Config, GPT2LMHeadModel
    c = GPT_CONFIGS[model]
    cfg = GPT2Config(n_embd=c["d"], n_layer=layers or c["layers"], n_head=max(1, c["d"] // 64),
                     vocab_size=c["vocab"], n_positions=c["ctx"], resid_pdrop=0.0, embd_pdrop=0.0,
                     attn_pdrop=0.0)
    torch.manual_seed(seed)
    m = GPT2LMHeadModel(cfg)
    return m.to(device)


def _shard_numel(params, world: int) -> int:
    """Per-rank flat shard numel FSDP2 builds for a group (dim-0 padded to world)."""
    n = 0
    for p in params:
        d0 = p.shape[0] if p.dim() > 0 else 1
        rest = p.numel() // max(d0, 1)
        n += math.ceil(d0 / world) * rest
    return n


def shard_model(model, mode: str, wspec: QuantSpec | None = None, gspec: QuantSpec | None = None,
                root_seed: int = 0, weight_levels=None, param_dtype=torch.bfloat16):
    """fully_shard every transformer block and the root; install QSDP comms if mode == 'qsdp'
    (``weight_levels``: a LevelTable when ``wspec.inner == "levels"``).  Both modes use the
    same mixed-precision policy: ``param_dtype`` all-gathered / computed parameters (bf16 by
    default; QSDP quantizes the fp32 master shards and writes that dtype), fp32 gradient
    reduce-scatter."""
    from torch.distributed.device_mesh import init_device_mesh
    from torch.distributed.fsdp import MixedPrecisionPolicy, fully_shard

    world = dist.get_world_size() if dist.is_initialized() else 1
    mesh = init_device_mesh("cuda", (world,))
    mp = MixedPrecisionPolicy(param_dtype=param_dtype, reduce_dtype=torch.float32)
    blocks = list(model.transformer.h)
    # one QSDP group collective carries a group's dense parameters: slots sized for the
    # largest group (codes padded per piece to 16 B, meta per piece to whole buckets)
    bucket = max((wspec or QuantSpec(8, 1024, "shift")).bucket, (gspec or QuantSpec(8, 1024)).bucket)

    min_bits = min((wspec or QuantSpec(8, 1024, "shift")).bits, (gspec or QuantSpec(8, 1024)).bits)

    def group_need(params):  # slot elements: quantized pieces + the full-precision ones' fp32 bytes
        dense = [p for p in params if p.dim() >= 2]
        raw = [p for p in params if p.dim() < 2]
        return (_shard_numel(dense, world) + len(dense) * (bucket + 16) +
                (_shard_numel(raw, world) + 4 * len(raw)) * 32 // min_bits)
    inner_ids = {id(p) for b in blocks for p in b.parameters()}
    max_shard = max([group_need(list(b.parameters())) for b in blocks] +
                    [group_need([p for p in model.parameters() if id(p) not in inner_ids])])
    for b in blocks:
        fully_shard(b, mesh=mesh, mp_policy=mp, reshard_after_forward=True)
    fully_shard(model, mesh=mesh, mp_policy=mp, reshard_after_forward=True)
    ctx = None
    if mode == "qsdp":
        from .fsdp import QSDPContext, apply_qsdp
        ctx = QSDPContext(max_shard, wspec or QuantSpec(8, 1024, "shift"),
                          gspec or QuantSpec(8, 1024, "uniform_stochastic"), root_seed=root_seed,
                          device=torch.device("cuda", torch.cuda.current_device()), weight_levels=weight_levels)
        apply_qsdp(blocks + [model], ctx, param_dtype)
    return ctx


def _tokens(gen, batch, seq, vocab, dev, learnable):
    if not learnable:
        return torch.randint(0, vocab, (batch, seq), device=dev, generator=gen)
    # learnable synthetic stream: t_{i+1} = (5 t_i + 3) mod 997, random start per row
    t0 = torch.randint(0, 997, (batch, 1), device=dev, generator=gen)
    out = [t0]
    for _ in range(seq - 1):
        out.append((out[-1] * 5 + 3) % 997)
    return torch.cat(out, dim=1)


def run_training(model, ctx, steps: int, batch: int, seq: int, warmup: int = 2, seed: int = 0,
                 lr: float = 6e-4, learnable: bool = False):
    """Train ``steps`` steps on synthetic tokens; returns (losses, ms per timed step)."""
    dev = torch.device("cuda", torch.cuda.current_device())
    rank = dist.get_rank() if dist.is_initialized() else 0
    opt = torch.optim.AdamW(model.parameters(), lr=lr, betas=(0.9, 0.95), weight_decay=0.0)
    gen = torch.Generator(device=dev)
    vocab = model.config.vocab_size
    losses, events = [], []
    stream = torch.cuda.current_stream(dev)
    for s in range(warmup + steps):
        gen.manual_seed(1000 * s + rank)
        tokens = _tokens(gen, batch, seq, vocab, dev, learnable)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        if ctx is not None:
            ctx.forward()
        with torch.autocast("cuda", dtype=torch.bfloat16):
            out = model(input_ids=tokens, labels=tokens)
        if ctx is not None:
            ctx.backward()
        out.loss.backward()
        opt.step()
        opt.zero_grad(set_to_none=True)
        if ctx is not None:
            ctx.next_step()
        ev1.record(stream)
        loss = out.loss.detach()
        if dist.is_initialized():
            dist.all_reduce(loss, op=dist.ReduceOp.AVG)
        if s >= warmup:
            events.append((ev0, ev1))
        losses.append(float(loss.item()))
    torch.cuda.synchronize(dev)
    times = torch.tensor([a.elapsed_time(b) for a, b in events], dtype=torch.float64, device=dev)
    if dist.is_initialized():  # device time, max over ranks
        dist.all_reduce(times, op=dist.ReduceOp.MAX)
    return losses, times.tolist()
