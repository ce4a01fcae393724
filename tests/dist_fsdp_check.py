"""FSDP2 + QSDP check (run under torchrun on >= 2 GPUs: FSDP2 issues no collectives
at world 1):

* comm parity -- one block group's QSDP all-gather / reduce-scatter on FSDP2's flat
  layout: dense weights bit-exact vs the oracle's per-parameter protocol; biases and
  LayerNorms gathered bit-identical to the unquantized FSDP2 all-gather and reduced
  bit-exactly as the reference averages them (sharded.py:359-371, 414-429);
* training -- a tiny GPT trained with QSDP comms tracks the unquantized FSDP2 run from
  the same initialisation (north_star: "a short training run tracks
  the reference loss curve")."""

import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2302_02390_b200.gpt_train import build_model, run_training, shard_model  # noqa: E402
from paper_2302_02390_b200.levels import learn_weight_levels  # noqa: E402
from paper_2302_02390_b200.quantize import QuantSpec  # noqa: E402


def comm_parity(rank, world, dev):
    """One group's QSDP all-gather / reduce-scatter against (a) the unquantized FSDP2
    collectives on the full-precision pieces (biases / norms: bit-identical) and (b) the
    oracle's protocol on the quantized pieces (dense weights: keys per parameter piece,
    sharded.py:323-433), with FSDP2's own flat layout and bf16 parameters."""
    import numpy as np
    from oracle import oracle as O
    from paper_2302_02390_b200.fsdp import QSDPAllGather, QSDPReduceScatter
    model = build_model("gpt-tiny", dev, seed=3)
    ctx = shard_model(model, "qsdp")
    group = dist.group.WORLD
    fails = 0
    layer = 1  # a transformer block: 4 dense weights, biases and two LayerNorms
    slots = ctx.layouts[layer]
    n = sum(s.numel for s in slots)
    ctx.step, ctx.phase = 7, 1
    masters = [s.fsdp_param._sharded_param_data for s in slots]
    inp = torch.cat([m.to(torch.bfloat16) for m in masters])  # FSDP2's copy-in
    out = torch.empty(world * n, dtype=torch.bfloat16, device=dev)
    QSDPAllGather(ctx, layer)(out, inp, group)
    ref = torch.empty_like(out)
    dist.all_gather_into_tensor(ref, inp)
    allm = [torch.empty(n, device=dev) for _ in range(world)]
    dist.all_gather(allm, torch.cat(masters))
    torch.cuda.synchronize()
    o, r = out.float().cpu().numpy(), ref.float().cpu().numpy()
    for s in slots:
        for q in range(world):
            a, b = q * n + s.offset, q * n + s.offset + s.numel
            if not s.dense:
                ok = np.array_equal(o[a:b], r[a:b])
            else:
                x = allm[q][s.offset:s.offset + s.numel].cpu().numpy()
                c, m, _ = O.quantize_segment(x, a, 1024, 8, 0, (0, 7, layer, 1, 0), 8)
                exp = torch.from_numpy(O.dequantize_segment(c, m, s.numel, 1024, 8).astype(np.float32))
                ok = np.array_equal(o[a:b], exp.to(torch.bfloat16).float().numpy())
            if not ok:
                fails += 1
                print(f"rank {rank} AG {s.name} dense={s.dense} shard {q}: mismatch", flush=True)
    g = torch.randn(world * n, device=dev, generator=torch.Generator(device=dev).manual_seed(100 + rank)) * 1e-3
    rs = torch.empty(n, device=dev)
    QSDPReduceScatter(ctx, layer)(rs, g, group, dist.ReduceOp.AVG)
    rs_ref = torch.empty(n, device=dev)
    dist.reduce_scatter_tensor(rs_ref, g.clone(), op=dist.ReduceOp.AVG)
    allg = [torch.empty_like(g) for _ in range(world)]
    dist.all_gather(allg, g)
    torch.cuda.synchronize()
    rsn, rrn = rs.cpu().numpy(), rs_ref.cpu().numpy()
    for s in slots:
        a, b = s.offset, s.offset + s.numel
        if not s.dense:  # the reference's acc + vals ... / P (fp64, ranks in order, one rounding)
            acc, mag = np.zeros(s.numel), np.zeros(s.numel)
            for p in range(world):
                v = allg[p][rank * n + a: rank * n + b].cpu().numpy().astype(np.float64)
                acc, mag = acc + v, mag + np.abs(v)
            ok = np.array_equal(rsn[a:b], (acc / world).astype(np.float32))
            if not ok:
                print(f"rank {rank} RS {s.name}: not the reference's ordered average", flush=True)
            # and within fp32 summation error of NCCL's AVG reduce-scatter (its own order)
            tol = world * np.finfo(np.float32).eps * mag / world
            if not np.all(np.abs(rsn[a:b].astype(np.float64) - rrn[a:b]) <= tol):
                ok = False
                print(f"rank {rank} RS {s.name}: beyond fp32 summation error of NCCL AVG", flush=True)
        else:
            acc = np.zeros(s.numel)
            for p in range(world):
                x = allg[p][rank * n + a: rank * n + b].cpu().numpy()
                c, m, _ = O.quantize_segment(x, rank * n + a, 1024, 8, 1, (0, 7, layer, 2, p), 8)
                acc = acc + O.dequantize_segment(c, m, s.numel, 1024, 8)
            ok = np.array_equal(rsn[a:b], (acc / world).astype(np.float32))
        if not ok:
            fails += 1
            print(f"rank {rank} RS {s.name} dense={s.dense}: mismatch", flush=True)
    if rank == 0:
        print(json.dumps({"comm_parity": {"group": layer, "params": [(s.name, s.numel, s.dense) for s in slots],
                                          "fails": fails}}), flush=True)
    ctx.close()
    return fails


def main():
    dist.init_process_group("nccl")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dev = torch.device("cuda", torch.cuda.current_device())
    steps = int(os.environ.get("QSDP_CHECK_STEPS", "30"))
    parity_fails = comm_parity(rank, world, dev)
    res = {}
    for mode in ("fsdp", "qsdp", "qsdp_w6_levels"):
        model = build_model("gpt-tiny", dev, seed=0)
        if mode == "qsdp_w6_levels":  # learned weight levels (paper's low-bit weights)
            table = learn_weight_levels([p for p in model.parameters() if p.dim() >= 2], 6)
            ctx = shard_model(model, "qsdp", wspec=QuantSpec(6, 1024, "levels"), weight_levels=table)
        else:
            ctx = shard_model(model, mode)
        losses, times = run_training(model, ctx, steps=steps, batch=8, seq=128, warmup=0, lr=1e-3,
                                     learnable=True)
        res[mode] = dict(losses=losses, calls=(ctx.calls if ctx else None))
        if ctx is not None:
            ctx.close()
        del model
    ok = True
    lf, lq, ll = res["fsdp"]["losses"], res["qsdp"]["losses"], res["qsdp_w6_levels"]["losses"]
    for curve in (lq, ll):
        if not (curve[-1] < curve[0] - 1.0):
            ok = False
        if abs(curve[-1] - lf[-1]) > 0.05 * lf[-1]:
            ok = False
    calls = res["qsdp"]["calls"]
    if world > 1 and (calls["allgather"] == 0 or calls["reducescatter"] == 0):
        ok = False  # (FSDP2 skips collectives entirely at world 1)
    if parity_fails:
        ok = False
    if rank == 0:
        print(json.dumps({"world": world, "fsdp_loss": [lf[0], lf[-1]], "qsdp_loss": [lq[0], lq[-1]],
                          "qsdp_w6_levels_loss": [ll[0], ll[-1]],
                          "calls": calls, "ok": ok}), flush=True)
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
