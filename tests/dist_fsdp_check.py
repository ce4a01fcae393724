"""FSDP2 + QSDP training check (run under torchrun, 1..N GPUs):
a tiny GPT trained with QSDP comms tracks the unquantized FSDP2 run from the
same initialisation (north_star: "a short training run
tracks the reference loss curve")."""

import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2302_02390_b200.gpt_train import build_model, run_training, shard_model  # noqa: E402
from paper_2302_02390_b200.levels import learn_weight_levels  # noqa: E402
from paper_2302_02390_b200.quantize import QuantSpec  # noqa: E402


def main():
    dist.init_process_group("nccl")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dev = torch.device("cuda", torch.cuda.current_device())
    steps = int(os.environ.get("QSDP_CHECK_STEPS", "30"))
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
    if rank == 0:
        print(json.dumps({"world": world, "fsdp_loss": [lf[0], lf[-1]], "qsdp_loss": [lq[0], lq[-1]],
                          "qsdp_w6_levels_loss": [ll[0], ll[-1]],
                          "calls": calls, "ok": ok}), flush=True)
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
