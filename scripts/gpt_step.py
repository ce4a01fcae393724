"""GPT training step on FSDP2: QSDP w8/g8 comms vs the unquantized FSDP2 baseline
(BASELINE.json configs[3]: "GPT 1.3B QSDP w8/g8 vs unquantized FSDP baseline").

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        scripts/gpt_step.py --model gpt-1.3b --batch 4 --seq 1024 --steps 8 [--out F.json]

Both modes use the identical setup (gpt_train.shard_model): random-init GPT, synthetic
tokens, one fully_shard group per block + root, bf16 parameters all-gathered / computed
(MixedPrecisionPolicy(param_dtype=bf16, reduce_dtype=fp32)), fp32 masters, AdamW.
Baseline = FSDP2's NCCL bf16 all-gather + fp32 reduce-scatter; QSDP = w8 weights / g8
gradients over the peer-memory communicator, biases and LayerNorms at full precision.
With N = 1 (no collectives at all) the step is the compute-only reference: exposed
communication at N = (step at N) - (step at 1), same per-GPU batch (weak scaling).
Device time per step with CUDA events, median over steps, max over ranks.
"""

import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_02390_b200.gpt_train import build_model, run_training, shard_model  # noqa: E402
from paper_2302_02390_b200.quantize import QuantSpec  # noqa: E402


def install_noop_comms(model):
    """Custom FSDP2 comms that move nothing (timing reference only: the step then runs FSDP2's
    copy-in / copy-out, compute and the sharded optimizer, without the collectives)."""
    from torch.distributed.fsdp import FSDPModule
    from torch.distributed.fsdp._fully_shard._fsdp_api import AllGather, ReduceScatter

    class NoAG(AllGather):
        def allocate(self, size, *, dtype, device):
            return torch.zeros(*size, dtype=dtype, device=device)

        def __call__(self, output_tensor, input_tensor, group, async_op=False):
            return None

    class NoRS(ReduceScatter):
        def allocate(self, size, *, dtype, device):
            return torch.zeros(*size, dtype=dtype, device=device)

        def __call__(self, output_tensor, input_tensor, group, op, async_op=False):
            return None

    for m in model.modules():
        if isinstance(m, FSDPModule):
            m.set_custom_all_gather(NoAG())
            m.set_custom_reduce_scatter(NoRS())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="gpt-1.3b")
    ap.add_argument("--batch", type=int, default=4)
    ap.add_argument("--seq", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--modes", default="fsdp,qsdp")
    ap.add_argument("--out", default="")
    ap.add_argument("--cprofile", action="store_true", help="rank 0: cProfile 2 more steps per mode (host hot spots)")
    ap.add_argument("--trace", default="", help="rank 0: torch.profiler chrome trace of 2 more steps per mode "
                                                "(file prefix)")
    a = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, world = dist.get_rank(), dist.get_world_size()
    res = {"model": a.model, "world": world, "batch_per_gpu": a.batch, "seq": a.seq, "steps": a.steps,
           "dtypes": "bf16 params / compute, fp32 masters + reduce-scatter", "data": "synthetic tokens"}
    for mode in a.modes.split(","):
        model = build_model(a.model, dev, seed=0)
        nparam = sum(p.numel() for p in model.parameters())
        ctx = shard_model(model, "fsdp" if mode == "nocomm" else mode, QuantSpec(8, 1024, "shift"),
                          QuantSpec(8, 1024, "uniform_stochastic"))
        if mode == "nocomm":  # compute-only reference at the same sharding: collectives replaced by no-ops
            install_noop_comms(model)
        losses, times = run_training(model, ctx, steps=a.steps, batch=a.batch, seq=a.seq, warmup=a.warmup)
        times = sorted(times)
        med = times[len(times) // 2]
        res[mode] = {"ms_per_step": round(med, 2), "steps_per_s": round(1e3 / med, 3),
                     "tokens_per_s": round(world * a.batch * a.seq / (med * 1e-3), 1),
                     "loss_first_last": [round(losses[0], 4), round(losses[-1], 4)],
                     "calls": ctx.calls if ctx is not None else None,
                     "host_ms_per_step_in_comm_hooks": ({k: round(1e3 * v / (a.steps + a.warmup), 3)
                                                         for k, v in ctx.host_s.items()} if ctx is not None else None)}
        if ctx is not None and ctx.capi_samples:
            import numpy as np
            v = np.array(ctx.capi_samples) * 1e6
            res[mode]["allgather_capi_us"] = {"median": round(float(np.median(v)), 1),
                                              "p90": round(float(np.percentile(v, 90)), 1),
                                              "max": round(float(v.max()), 1), "n": int(v.size)}
        res["params"] = nparam
        if a.trace and rank == 0:
            from torch.profiler import ProfilerActivity, profile
            with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
                run_training(model, ctx, steps=2, batch=a.batch, seq=a.seq, warmup=0)
            prof.export_chrome_trace(f"{a.trace}_{mode}.json")
        elif a.trace:
            run_training(model, ctx, steps=2, batch=a.batch, seq=a.seq, warmup=0)
        if a.cprofile:
            import cProfile
            import pstats
            pr = cProfile.Profile()
            pr.enable()
            run_training(model, ctx, steps=2, batch=a.batch, seq=a.seq, warmup=0)
            pr.disable()
            if rank == 0:
                print(f"== cProfile {mode} (2 steps)", flush=True)
                pstats.Stats(pr).sort_stats("tottime").print_stats(25)
        if ctx is not None:
            ctx.close()
        del model
        torch.cuda.empty_cache()
    if "fsdp" in res and "qsdp" in res:
        res["qsdp_speedup"] = round(res["fsdp"]["ms_per_step"] / res["qsdp"]["ms_per_step"], 4)
    if "nocomm" in res:  # exposed communication = step - compute-only step (same sharding)
        for m in ("fsdp", "qsdp"):
            if m in res:
                res[m]["exposed_comm_ms"] = round(res[m]["ms_per_step"] - res["nocomm"]["ms_per_step"], 2)
    if rank == 0:
        print(json.dumps(res), flush=True)
        if a.out:
            json.dump(res, open(a.out, "w"), indent=1)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
