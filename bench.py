#!/usr/bin/env python
"""QSDP communication hot-path benchmark (driver contract: one JSON line).

Metric (BASELINE.json): quantized all-gather + reduce-scatter effective GB/s.
Workload (configs[1]): GPT-2 small (125M) dense parameter groups, QSDP w8/g8,
bucket 1024, synthetic N(0, 0.02^2) weights and N(0, 1e-3^2) gradients.  One
step = one training step's QSDP traffic: for every FSDP group (root + 12
blocks) a forward all-gather (phase 0), then in reverse order a backward
re-gather (phase 1) and a gradient reduce-scatter (phase 2) -- the call order
of forward_layer/backward_layer (pkg/src/qsdp/sharded.py:437-469).

effective GB/s (nccl-tests algbw convention on the fp32 tensor):
per rank 4*N bytes per collective, 3 collectives per group; ``value`` is the
whole-job aggregate (sum over ranks), scaling "weak" (each rank dequantizes
the full model per gather whatever N is).

    python bench.py [--gpus N --steps K --warmup W --model gpt2-125m --wbits 8 --gbits 8 --bucket 1024]
    python bench.py --impl reference ...   # the reference algorithm on the host CPU (oracle port)
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
           0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
           0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


def pin_to_gpu_numa(local: int) -> None:
    """Run this rank on the CPUs next to its GPU (the PCIe root's NUMA node), so the pinned host
    buffers of the e2e step are allocated in local memory.  No-op where sysfs does not say."""
    import torch
    try:
        p = torch.cuda.get_device_properties(local)
        bus = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
        spec = open(f"/sys/bus/pci/devices/{bus}/local_cpulist").read().strip()
        cpus = set()
        for part in spec.split(","):
            a, _, b = part.partition("-")
            cpus.update(range(int(a), int(b or a) + 1))
        cpus &= os.sched_getaffinity(0)
        if cpus:
            os.sched_setaffinity(0, cpus)
    except Exception:
        pass


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--model", default="gpt2-125m")
    ap.add_argument("--wbits", type=int, default=8)
    ap.add_argument("--gbits", type=int, default=8)
    ap.add_argument("--bucket", type=int, default=1024)
    ap.add_argument("--out-dtype", default="f32", choices=["f32", "bf16"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--check-e2e", action="store_true", help="verify the e2e step's results once")
    ap.add_argument("--no-gpt", action="store_true")
    ap.add_argument("--no-levels", action="store_true", help="skip the learned-levels kernel timings")
    ap.add_argument("--serial", action="store_true",
                    help="one stream for every collective (default: FSDP2's schedule, RS on its own stream/comm)")
    ap.add_argument("--inflight", type=int, default=16,
                    help="collectives of one kind in flight (streams + communicators per kind; the prefetch depth). "
                         "At N>1 deeper pipelines hide the barrier waits and NVLink pushes (N=4: 2 -> 8 in flight "
                         "+13%%, N=2: 8 -> 16 +3.5%%); N=1 +1.5%% from 8 to 16")
    ap.add_argument("--fwd-ag-sms", type=int, default=0, help="SM budget of the forward all-gathers (0 = all)")
    ap.add_argument("--bwd-ag-sms", type=int, default=0, help="SM budget of the backward all-gathers (0 = all)")
    ap.add_argument("--rs-sms", type=int, default=0, help="SM budget of the reduce-scatters (0 = all)")
    ap.add_argument("--fwd-ag-ctas", type=int, default=1,
                    help="quantizer CTAs per SM, forward all-gathers (0 = occupancy, 2 for this kernel). One: "
                         "two in-flight all-gathers share every SM, one's ramp / tail under the other's "
                         "steady state (N=1 +2%%, DESIGN §17)")
    ap.add_argument("--bwd-ag-ctas", type=int, default=1, help="quantizer CTAs per SM, backward all-gathers")
    ap.add_argument("--rs-ctas", type=int, default=0, help="quantizer CTAs per SM, reduce-scatters")
    ap.add_argument("--rs-priority", type=int, default=0,
                    help="CUDA stream priority of the reduce-scatter streams (-1 = high: their CTAs are "
                         "dispatched before queued all-gather CTAs)")
    ap.add_argument("--trace", default="", help="write the GPU timeline of one step replay (CUPTI via "
                    "torch.profiler: every kernel's start / end / stream) and its overlap summary to this JSON file")
    ap.add_argument("--gpt-steps", type=int, default=8)
    ap.add_argument("--gpt-batch", type=int, default=8, help="sequences per GPU")
    ap.add_argument("--gpt-seq", type=int, default=1024)
    return ap.parse_args()


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index, self.samples, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 3:
                try:
                    self.samples.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
                except ValueError:
                    pass

    def __exit__(self, *a):
        if not self.samples:  # timed region shorter than the sampling period: take one reading now
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                      "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=20)
                parts = [p.strip() for p in out.stdout.strip().split(",")]
                self.samples.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
            except Exception:
                pass
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sms = sorted(s[0] for s in self.samples)
        reasons = set()
        for _, _, mask in self.samples:
            for bit, name in REASONS.items():
                if mask & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": sms[len(sms) // 2], "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": sorted(reasons), "samples": len(sms)}


# ---------------------------------------------------------------------------
# CPU reference arm: the reference algorithm (oracle port of pkg/src/qsdp) on host cores.
# ---------------------------------------------------------------------------

def cpu_protocol_step(O, full_w, grads, P, wbits, gbits, bucket, step, threads):
    """AG(fwd) + AG(bwd) + RS over P virtual ranks, as sharded.py:323-433."""
    O.gather(full_w, P, bucket, wbits, 0, step, 1, 0, threads)
    O.gather(full_w, P, bucket, wbits, 0, step, 1, 1, threads)
    O.reduce_scatter(grads, bucket, gbits, 0, step, 1, threads)


def cpu_sample(model, world):
    import numpy as np
    from paper_2302_02390_b200.gpt import dense_groups
    g = dense_groups(model)[1]  # first transformer block group
    n = max(1 << 18, g.numel // max(1, world))
    rng = np.random.default_rng(0)
    w = (rng.standard_normal(n) * 0.02).astype(np.float32)
    grads = [(np.random.default_rng(1 + p).standard_normal(n) * 1e-3).astype(np.float32) for p in range(world)]
    return g, n, w, grads


def run_cpu_baseline(args, world, min_seconds=10.0):
    from oracle import oracle as O
    threads = len(os.sched_getaffinity(0))
    _, n, w, grads = cpu_sample(args.model, world)
    reps, t0 = 0, time.perf_counter()
    while True:
        cpu_protocol_step(O, w, grads, world, args.wbits, args.gbits, args.bucket, reps, threads)
        reps += 1
        el = time.perf_counter() - t0
        if el >= min_seconds or reps >= 50:
            break
    value = world * 12.0 * n * reps / el / 1e9
    return {"value": round(value, 4), "unit": "GB/s", "cores": threads, "kind": "port",
            "sample": f"{reps} x [AG fwd + AG bwd + RS] of {n} elements (first {args.model} block group, "
                      f"P={world} virtual ranks), w{args.wbits}/g{args.gbits} bucket {args.bucket}, "
                      f"{el:.1f} s wall, C oracle (oracle/qsdp_oracle.c) on {threads} threads"}


def reference_workload(model, world):
    """The B200 arm's step workload on the host: every dense FSDP group's weights and P virtual
    ranks' gradients (rank p's gradient is a rotation of one N(0, 1e-3^2) draw -- the timing
    does not depend on the values).  The simulated RS does P x the quantization work of P = 1
    (every rank quantizes its whole gradient), so for world > 2 the step is a bounded sample
    -- the leading groups up to 4/(2+P) of the parameters -- to keep the run within minutes."""
    import numpy as np
    from paper_2302_02390_b200.gpt import dense_groups
    groups = dense_groups(model)
    if world > 2:
        total, keep, acc = sum(g.numel for g in groups), [], 0
        for g in groups:
            if acc >= total * 4.0 / (2 + world):
                break
            keep.append(g)
            acc += g.numel
        groups = keep
    rng = np.random.default_rng(0)
    work = []
    for g in groups:
        w = (rng.standard_normal(g.numel, dtype=np.float32) * np.float32(0.02))
        base = rng.standard_normal(g.numel, dtype=np.float32) * np.float32(1e-3)
        grads = [np.roll(base, 7919 * p) for p in range(world)]
        work.append((w, grads))
    return groups, work


def run_reference(args):
    """The reference's CPU implementation of the path (the C oracle port of sharded.py:323-433 /
    quantize.py / wire.py, every host thread) on the B200 arm's own config: per step, AG fwd +
    AG bwd + RS over every dense group of the model at P = world virtual ranks (the reference is
    a single-process simulation of all P ranks)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    from oracle import oracle as O
    threads = len(os.sched_getaffinity(0))
    from paper_2302_02390_b200.gpt import dense_groups
    all_groups = dense_groups(args.model)
    groups, work = reference_workload(args.model, world)
    n_total = sum(g.numel for g in groups)
    full = len(groups) == len(all_groups)
    warm = min(args.warmup, 1)  # host code: one warm-up step pages the arrays in

    def step(s):
        for li, (w, grads) in enumerate(work):
            O.gather(w, world, args.bucket, args.wbits, 0, s, li, 0, threads)
            O.gather(w, world, args.bucket, args.wbits, 0, s, li, 1, threads)
            O.reduce_scatter(grads, args.bucket, args.gbits, 0, s, li, threads)

    for s in range(warm):
        step(s)
    t0 = time.perf_counter()
    for s in range(args.steps):
        step(warm + s)
    el = time.perf_counter() - t0
    value = world * 12.0 * n_total * args.steps / el / 1e9
    line = {
        "impl": "reference", "metric": "quantized all-gather+reduce-scatter effective GB/s", "value": round(value, 4),
        "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": warm,
        "ms_per_step": round(el / args.steps * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(args, world, len(all_groups), sum(g.numel for g in all_groups)),
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": threads, "kind": "port",
                         "sample": ("the full step" if full else f"a bounded sample of the step (the leading "
                                                                   f"{len(groups)} of {len(all_groups)} groups)")
                                   + f": AG fwd + AG bwd + RS over {n_total} elements at P={world} virtual "
                                     f"ranks, oracle/qsdp_oracle.c on {threads} threads"},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def trace_step(g, flush, path):
    """Timeline of one step-graph replay (after an L2 flush): CUPTI kernel records through
    torch.profiler, reduced to per-kernel intervals and the overlap between streams
    (no nsys in this image)."""
    import tempfile

    import torch
    from torch.profiler import ProfilerActivity, profile
    flush.fill_(7)
    torch.cuda.synchronize()
    if not path:
        g.replay()
        torch.cuda.synchronize()
        return
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        g.replay()
        torch.cuda.synchronize()
    with tempfile.NamedTemporaryFile(suffix=".json") as f:
        prof.export_chrome_trace(f.name)
        tr = json.load(open(f.name))
    ks = [e for e in tr.get("traceEvents", []) if e.get("ph") == "X" and e.get("cat") == "kernel"]
    ks.sort(key=lambda e: e["ts"])
    t0 = ks[0]["ts"] if ks else 0.0
    rec = [{"name": e["name"][:90], "stream": e.get("args", {}).get("stream"), "start_us": round(e["ts"] - t0, 2),
            "end_us": round(e["ts"] + e["dur"] - t0, 2)} for e in ks]
    # union of busy time, and the time with >= 2 kernels running
    pts = sorted([(r["start_us"], 1) for r in rec] + [(r["end_us"], -1) for r in rec])
    busy = multi = 0.0
    depth, last = 0, None
    for t, d in pts:
        if last is not None and depth > 0:
            busy += t - last
            if depth > 1:
                multi += t - last
        depth += d
        last = t
    summ = {"kernels": len(rec), "span_us": round(rec[-1]["end_us"], 2) if rec else 0.0,
            "sum_kernel_us": round(sum(r["end_us"] - r["start_us"] for r in rec), 2), "busy_us": round(busy, 2),
            "overlapped_us": round(multi, 2), "streams": sorted({str(r["stream"]) for r in rec}),
            "how": "torch.profiler (CUPTI) of one replay of the timed step graph; times relative to the first kernel"}
    json.dump({"summary": summ, "kernels": rec}, open(path, "w"), indent=1)
    print(f"trace: {summ}", file=sys.stderr, flush=True)


def bench_config(args, world, ngroups, n_total):
    """The workload both arms report (the reference arm runs the same step on the host)."""
    return {"workload": f"{args.model} QSDP w{args.wbits}/g{args.gbits} bucket {args.bucket}: per step "
                        f"AG fwd + AG bwd + RS over {ngroups} FSDP groups ({n_total} dense params)",
            "out_dtype": args.out_dtype, "quantizer_input": "f32", "arithmetic": "f64 (bit-exact)",
            "parallelism": f"qsdp{world}", "convention": "sum over ranks of 4*N per collective / time",
            "inflight": args.inflight, "ag_ctas_per_sm": [args.fwd_ag_ctas, args.bwd_ag_ctas]}


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------

def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_2302_02390_b200 import _lib
    from paper_2302_02390_b200.comm import QSDPComm, plan_segments
    from paper_2302_02390_b200.gpt import dense_groups
    from paper_2302_02390_b200.quantize import (QuantSpec, SegmentKey, advance_counter, codes_bytes,
                                                dequant_accumulate, dequantize_segments, num_buckets,
                                                quantize_segments)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pin_to_gpu_numa(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    _lib.lib()

    wspec = QuantSpec(args.wbits, args.bucket, "shift")
    gspec = QuantSpec(args.gbits, args.bucket, "uniform_stochastic")
    out_dt = torch.float32 if args.out_dtype == "f32" else torch.bfloat16
    osz = 4 if out_dt == torch.float32 else 2
    groups = dense_groups(args.model)
    N_total = sum(g.numel for g in groups)
    pad = args.bucket if args.bucket % 8 == 0 else 1

    # ---- synthetic state, resident in HBM for `value` ----
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    state = []
    max_seg = 0
    for g in groups:
        segs = plan_segments(g.numel, world, pad)
        max_seg = max(max_seg, max(n for _, n in segs))
        s, n = segs[rank]
        st = dict(g=g, segs=segs, n=n)
        st["shard"] = torch.randn(max(n, 1), generator=gen, device=dev)[:n].mul_(0.02)
        st["grad"] = torch.randn(g.numel, generator=gen, device=dev).mul_(1e-3)
        st["full"] = torch.empty(g.numel, dtype=out_dt, device=dev)
        st["gshard"] = torch.empty(max(n, 1), dtype=torch.float32, device=dev)
        st["wq"] = (torch.empty(codes_bytes(g.numel, wspec) + 16, dtype=torch.uint8, device=dev),
                    torch.empty((num_buckets(g.numel, args.bucket), 3), dtype=torch.float32, device=dev))
        st["gq"] = (torch.empty(codes_bytes(g.numel, gspec) + 16, dtype=torch.uint8, device=dev),
                    torch.empty((num_buckets(g.numel, args.bucket), 3), dtype=torch.float32, device=dev))
        state.append(st)
    flush = torch.empty(64 << 20, dtype=torch.int32, device=dev)  # 256 MB > 126 MB L2
    step_ctr = torch.zeros(1, dtype=torch.int64, device=dev)
    # FSDP2's schedule (fsdp.QSDPContext): all-gathers on one stream, reduce-scatters on their
    # own stream with their own communicator, RS(i) after AG(i)'s backward re-gather, overlapping
    # AG(i-1).  --inflight K keeps K collectives of each kind in flight (K streams and
    # communicators per kind, round robin: FSDP2's prefetch depth), so one collective's tail
    # overlaps the next one's ramp; --*-sms split the SMs between the overlapping kinds.
    K = max(1, args.inflight)
    stream = torch.cuda.current_stream(dev)
    ag_comms = [QSDPComm(max_seg, wspec, gspec, device=dev) for _ in range(K)]
    rs_comms = ag_comms if args.serial else [QSDPComm(max_seg, wspec, gspec, device=dev) for _ in range(K)]
    for c in set(ag_comms + rs_comms):
        c.set_step_source(step_ctr)
    comm, rs_comm = ag_comms[0], rs_comms[0]
    # all-gather slot 0 runs on the issuing stream (the capture stream inside a graph)
    ag_side = [torch.cuda.Stream(device=dev) for _ in range(K - 1)]
    rs_side = [torch.cuda.Stream(device=dev, priority=args.rs_priority) for _ in range(K)]
    rs_stream = rs_side[0]

    # ---- the step as a list of launches (kind, bytes, fn) ----
    kinds = ("K1_quantize_shift", "K3_dequantize", "K2_quantize_stochastic", "K4_dequant_accumulate")

    def local_launches():
        """World 1: the comm's kernels through the batched API (same kernels, per-kernel timing)."""
        L = []

        def ag(st, gi, phase):
            n = st["g"].numel
            cb = codes_bytes(n, wspec) + 12 * num_buckets(n, args.bucket)
            L.append((kinds[0], 4 * n + cb, lambda: quantize_segments(
                [(st["shard"], 0, SegmentKey(0, 0, gi, phase, 0))], wspec, out=[st["wq"]], step_src=step_ctr)))
            L.append((kinds[1], cb + osz * n, lambda: dequantize_segments(
                [(st["wq"][0], st["wq"][1], n, st["full"])], wspec, out_dt)))

        def rs(st, gi):
            n = st["g"].numel
            cb = codes_bytes(n, gspec) + 12 * num_buckets(n, args.bucket)
            L.append((kinds[2], 4 * n + cb, lambda: quantize_segments(
                [(st["grad"], 0, SegmentKey(0, 0, gi, 2, 0))], gspec, out=[st["gq"]], step_src=step_ctr)))
            L.append((kinds[3], cb + 4 * n, lambda: dequant_accumulate(
                [(st["gq"][0], st["gq"][1])], n, gspec, 1, dtype=torch.float32, out=st["gshard"])))

        for gi, st in enumerate(state):
            ag(st, gi, 0)
        for gi in range(len(state) - 1, -1, -1):
            ag(state[gi], gi, 1)
            rs(state[gi], gi)
        return L

    def comm_launches():
        """The step's collectives: (kind, launches, fn, slot, after): slot = the stream /
        communicator index within the kind; `after` = index of the launch it must follow."""
        L = []
        per = 3 if world > 1 else 2  # quantize (+ barrier) + dequant
        j = 0
        for gi, st in enumerate(state):
            c = ag_comms[j % K]
            L.append(("AG", per, lambda st=st, gi=gi, c=c: (c.set_sm_budget(args.fwd_ag_sms),
                                                           c.set_ctas_per_sm(args.fwd_ag_ctas), c.all_gather(
                st["shard"], st["segs"], SegmentKey(0, 0, gi, 0, 0), st["full"])), ("ag", j % K), None))
            j += 1
        r = 0
        for gi in range(len(state) - 1, -1, -1):
            st = state[gi]
            c = ag_comms[j % K]
            L.append(("AG", per, lambda st=st, gi=gi, c=c: (c.set_sm_budget(args.bwd_ag_sms),
                                                           c.set_ctas_per_sm(args.bwd_ag_ctas), c.all_gather(
                st["shard"], st["segs"], SegmentKey(0, 0, gi, 1, 0), st["full"])), ("ag", j % K), None))
            j += 1
            c = rs_comms[r % K]
            L.append(("RS", per, lambda st=st, gi=gi, c=c: (c.set_sm_budget(args.rs_sms),
                                                           c.set_ctas_per_sm(args.rs_ctas), c.reduce_scatter(
                st["grad"], st["segs"], SegmentKey(0, 0, gi, 2, rank), st["gshard"])),
                ("ag" if args.serial else "rs", (r if args.serial else r) % K), len(L) - 1))
            r += 1
        return L

    def issue(launches):
        """Issue a step's collectives on their streams (forked from and joined to the current stream)."""
        main = torch.cuda.current_stream(dev)
        ag_streams = [main] + ag_side
        rs_streams = ag_streams if args.serial else rs_side
        used = {id(main)}
        start = torch.cuda.Event()
        start.record(main)
        done = {}
        for idx, (_, _, fn, (kind, slot), after) in enumerate(launches):
            s_ = (ag_streams if kind == "ag" else rs_streams)[slot]
            if id(s_) not in used:
                s_.wait_event(start)
                used.add(id(s_))
            if after is not None:
                s_.wait_event(done[after])
            with torch.cuda.stream(s_):
                fn()
            ev = torch.cuda.Event()
            ev.record(s_)
            done[idx] = ev
        for s_ in set(ag_streams + rs_streams):
            if s_ is not main and id(s_) in used:
                main.wait_stream(s_)

    # `value` times the product path (the communicator); the per-kernel roofline graphs replay
    # the same kernels through the batch API.
    launches = comm_launches()
    klaunches = local_launches() if world == 1 else []
    per_coll = 3 if world > 1 else 1  # world 1: one quantizer launch with the fused dequant
    n_launch = len(launches) * per_coll + 1  # + step counter (replaced by the captured graph's kernel-node count)

    def run_step(sel=None):
        if sel is None:
            issue(launches)
            advance_counter(step_ctr)
        else:
            for kind, _, fn in klaunches:
                if kind == sel:
                    fn()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def capture(fn, keep=False):
        try:
            g = torch.cuda.CUDAGraph(keep_graph=keep)
        except TypeError:
            g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        return g

    def kernel_nodes(g):
        """Kernel nodes of a captured step graph (every one is a launch of this library's kernels:
        the step holds only the communicator's collectives and the step-counter update)."""
        try:
            from cuda.bindings import runtime as rt
            h = rt.cudaGraph_t(init_value=g.raw_cuda_graph())
            err, _, n = rt.cudaGraphGetNodes(h, 0)
            err, nodes, n = rt.cudaGraphGetNodes(h, n)
            if err != rt.cudaError_t.cudaSuccess:
                return None
            return sum(1 for nd in nodes
                       if rt.cudaGraphNodeGetType(nd)[1] == rt.cudaGraphNodeType.cudaGraphNodeTypeKernel)
        except Exception:
            return None

    def time_graph(g, reps, flush_between=True):
        ev = []
        for r in range(reps):
            if flush_between:
                flush.fill_(r)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            g.replay()
            b.record(stream)
            ev.append((a, b))
        return ev

    for _ in range(args.warmup):
        run_step()
    barrier()
    g_step = capture(run_step, keep=True)
    nodes = kernel_nodes(g_step)
    if nodes is not None:
        n_launch = nodes
    for _ in range(args.warmup):  # warm the graph itself
        g_step.replay()
    barrier()
    with ClockSampler(local) as clocks:
        barrier()
        ev = time_graph(g_step, args.steps)
        barrier()
    ms = sum(a.elapsed_time(b) for a, b in ev)
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    if args.trace:  # every rank replays (the collectives' barriers need all of them); rank 0 records
        barrier()
        trace_step(g_step, flush, args.trace if rank == 0 else "")
        barrier()
    value = world * 12.0 * N_total / (ms_step * 1e-3) / 1e9

    # ---- roofline of the dominant kernel: per-kind graphs timed with CUDA events ----
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    kernels, roofline = {}, None
    if world == 1:
        for k in kinds:
            nb = sum(x[1] for x in klaunches if x[0] == k)
            cnt = sum(1 for x in klaunches if x[0] == k)
            gk = capture(lambda k=k: run_step(k))
            gk.replay()
            torch.cuda.synchronize(dev)
            evk = time_graph(gk, args.steps)
            torch.cuda.synchronize(dev)
            tk = sum(a.elapsed_time(b) for a, b in evk) / args.steps
            kernels[k] = {"ms_per_step": round(tk, 4), "launches_per_step": cnt, "avg_launch_us": round(tk / cnt * 1e3, 2),
                          "gbs": round(nb / (tk * 1e-3) / 1e9, 1), "share_of_step": round(tk / ms_step, 4),
                          "bytes_per_step": nb}
        # The step's own launches: at world 1 each collective is ONE quantizer launch with the fused
        # dequant epilogue (AG: K1 + K3 of the own shard; RS: K2 + K4's 0.0 + v), so the roofline is
        # taken over those kinds, timed the same way; the four standalone kernels (the N > 1 path and
        # the batch API) stay listed as kernels_unfused.
        osz = 4 if out_dt == torch.float32 else 2
        fused_kinds = {}
        # the kernels' own throughput: serial on one stream, at full occupancy (the step pairs its
        # in-flight all-gathers at --*-ag-ctas CTAs per SM; that schedule is timed separately below)
        sched = (args.fwd_ag_ctas, args.bwd_ag_ctas, args.rs_ctas)
        args.fwd_ag_ctas = args.bwd_ag_ctas = args.rs_ctas = 0
        for kind, sel in (("AG_K1_fused_dequant", "AG"), ("RS_K2_fused_dequant", "RS")):
            fns = [x[2] for x in launches if x[0] == sel]  # serial on one stream: the kernels' own throughput
            gk = capture(lambda fns=fns: [f() for f in fns], keep=True)
            cnt = kernel_nodes(gk) or len(fns)
            if cnt != len(fns):  # not fused for this config: keep the standalone breakdown
                fused_kinds = {}
                break
            gk.replay()
            torch.cuda.synchronize(dev)
            evk = time_graph(gk, args.steps)
            torch.cuda.synchronize(dev)
            tk = sum(a.elapsed_time(b) for a, b in evk) / args.steps
            reps = 2 if sel == "AG" else 1
            nb = reps * sum(4 * st["n"] + (osz if sel == "AG" else 4) * st["n"] + 12 * num_buckets(st["n"], args.bucket)
                            for st in state)
            fused_kinds[kind] = {"ms_per_step": round(tk, 4), "launches_per_step": cnt,
                                 "avg_launch_us": round(tk / cnt * 1e3, 2), "gbs": round(nb / (tk * 1e-3) / 1e9, 1),
                                 "share_of_step": round(tk / ms_step, 4), "bytes_per_step": nb,
                                 "bytes_per_element": f"4 in + {osz if sel == 'AG' else 4} out + 12/{args.bucket} meta "
                                                      "(no codes: world 1 has no reader)"}
        args.fwd_ag_ctas, args.bwd_ag_ctas, args.rs_ctas = sched
        if fused_kinds and any(sched):  # the same serial graphs at the step's CTA caps
            for kind, sel in (("AG_K1_fused_dequant", "AG"), ("RS_K2_fused_dequant", "RS")):
                fns = [x[2] for x in launches if x[0] == sel]
                gk = capture(lambda fns=fns: [f() for f in fns], keep=True)
                gk.replay()
                torch.cuda.synchronize(dev)
                evk = time_graph(gk, args.steps)
                torch.cuda.synchronize(dev)
                tk = sum(a.elapsed_time(b) for a, b in evk) / args.steps
                fused_kinds[kind]["gbs_at_step_ctas"] = round(fused_kinds[kind]["bytes_per_step"] / (tk * 1e-3) / 1e9, 1)
        kernels_unfused = None
        if fused_kinds:
            kernels_unfused, kernels = kernels, fused_kinds
        dom = max(kernels, key=lambda k: kernels[k]["ms_per_step"])
        ach = kernels[dom]["gbs"]
        traffic = None
        try:
            tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
            traffic = tr.get(args.model, {}).get(dom)
        except Exception:
            pass
        roofline = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": hbm_peak, "unit": "GB/s",
                    "frac": round(ach / hbm_peak, 4), "traffic": traffic, "peak_source": peak_src,
                    "bytes_per_launch": round(kernels[dom]["bytes_per_step"] / kernels[dom]["launches_per_step"]),
                    "method": "algorithmic bytes / CUDA-event time of that kernel's launches (graph of one step's "
                              "launches of the kind, serial, full occupancy, L2 flushed between replays)",
                    "frac_by_kernel": {k: round(v["gbs"] / hbm_peak, 4) for k, v in kernels.items()}}
        if "K2" in dom:
            roofline["note"] = ("K2 is integer-issue bound: one exact 128-bit PCG64 step per element "
                                "(numpy's bucket_rng stream, DESIGN.md section 5)")
        if "gbs_at_step_ctas" in kernels[dom]:
            roofline["frac_at_step_ctas"] = {k: round(v["gbs_at_step_ctas"] / hbm_peak, 4) for k, v in kernels.items()
                                             if "gbs_at_step_ctas" in v}
        if kernels_unfused is not None:
            roofline["frac_by_kernel_unfused"] = {k: round(v["gbs"] / hbm_peak, 4) for k, v in kernels_unfused.items()}

    # ---- learned-levels kernels on the same weight groups (world 1) ----
    levels = None
    if world == 1 and not args.no_levels:
        from paper_2302_02390_b200.levels import LevelTable, dequantize_levels, learn_levels, quantize_levels_segments
        lspec = QuantSpec(args.wbits, args.bucket, "levels")
        u = torch.rand(1 << 18, generator=gen, device=dev, dtype=torch.float64)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        table = learn_levels(u, LevelTable.uniform(args.wbits))
        b.record(stream)
        torch.cuda.synchronize(dev)
        learn_ms = a.elapsed_time(b)
        for st in state:
            st["lq"] = (torch.empty(codes_bytes(st["g"].numel, lspec) + 16, dtype=torch.uint8, device=dev),
                        torch.empty((num_buckets(st["g"].numel, args.bucket), 3), dtype=torch.float32, device=dev))
        lbytes = {"LQ_quantize_levels": sum(4 * st["g"].numel + codes_bytes(st["g"].numel, lspec)
                                            + 12 * num_buckets(st["g"].numel, args.bucket) for st in state),
                  "LD_dequantize_levels": sum(osz * st["g"].numel + codes_bytes(st["g"].numel, lspec)
                                              + 12 * num_buckets(st["g"].numel, args.bucket) for st in state)}

        def lq_all():
            for st in state:
                quantize_levels_segments([st["shard"]], lspec, table, out=[st["lq"]])

        def ld_all():
            for st in state:
                dequantize_levels(st["lq"][0], st["lq"][1], st["g"].numel, lspec, table, dtype=out_dt, out=st["full"])

        levels = {"table": f"{1 << args.wbits} levels learned (Alg. 2) on 2^18 uniform values",
                  "learn_levels_values_per_s": round(u.numel() / (learn_ms * 1e-3), 1)}
        for name, fn in (("LQ_quantize_levels", lq_all), ("LD_dequantize_levels", ld_all)):
            fn()
            gk = capture(fn)
            gk.replay()
            torch.cuda.synchronize(dev)
            evk = time_graph(gk, args.steps)
            torch.cuda.synchronize(dev)
            tk = sum(a.elapsed_time(b) for a, b in evk) / args.steps
            levels[name] = {"ms_per_pass": round(tk, 4), "gbs": round(lbytes[name] / (tk * 1e-3) / 1e9, 1),
                            "frac_of_hbm_peak": round(lbytes[name] / (tk * 1e-3) / 1e9 / hbm_peak, 4),
                            "bytes_per_pass": lbytes[name], "launches_per_pass": len(state)}

    # ---- counter-based noise (QSDP_NOISE_PHILOX4x64): K1 / K2 with numpy's Philox4x64-10 ----
    philox = None
    if world == 1 and not args.no_levels:
        pws = QuantSpec(args.wbits, args.bucket, "shift", "philox")
        pgs = QuantSpec(args.gbits, args.bucket, "uniform_stochastic", "philox")

        def pq_w():
            for gi, st in enumerate(state):
                quantize_segments([(st["shard"], 0, SegmentKey(0, 0, gi, 0, 0))], pws, out=[st["wq"]])

        def pq_g():
            for gi, st in enumerate(state):
                quantize_segments([(st["grad"], 0, SegmentKey(0, 0, gi, 2, 0))], pgs, out=[st["gq"]])

        pbytes = {"K1_quantize_shift_philox": sum(4 * st["n"] + codes_bytes(st["n"], pws)
                                                  + 12 * num_buckets(st["n"], args.bucket) for st in state),
                  "K2_quantize_stochastic_philox": sum(4 * st["g"].numel + codes_bytes(st["g"].numel, pgs)
                                                       + 12 * num_buckets(st["g"].numel, args.bucket) for st in state)}
        philox = {"noise": "np.random.Generator(np.random.Philox(SeedSequence(key))): Philox4x64-10, counter-based "
                           "(one 10-round block per 4 draws); K1 on the TMA32 path (one draw per bucket), K2 on the "
                           "TMA32 octet path (two blocks per lane-octet; team kernels for other bucket shapes)"}
        for name, fn in (("K1_quantize_shift_philox", pq_w), ("K2_quantize_stochastic_philox", pq_g)):
            fn()
            gk = capture(fn)
            gk.replay()
            torch.cuda.synchronize(dev)
            evk = time_graph(gk, args.steps)
            torch.cuda.synchronize(dev)
            tk = sum(a.elapsed_time(b) for a, b in evk) / args.steps
            philox[name] = {"ms_per_pass": round(tk, 4), "gbs": round(pbytes[name] / (tk * 1e-3) / 1e9, 1),
                            "frac_of_hbm_peak": round(pbytes[name] / (tk * 1e-3) / 1e9 / hbm_peak, 4),
                            "bytes_per_pass": pbytes[name], "launches_per_pass": len(state)}

    # ---- GPU wire codec over the step's weight messages (world 1) ----
    wire = None
    if world == 1 and not args.no_levels:
        from paper_2302_02390_b200.wire import decode_segment, encode_segment
        for gi, st in enumerate(state):  # fill the weight slots with real codes first
            quantize_segments([(st["shard"], 0, SegmentKey(0, 0, gi, 0, 0))], wspec, out=[st["wq"]])
        msgs = [encode_segment(st["wq"][0], st["wq"][1], st["g"].numel, wspec) for st in state]
        mbytes = sum(m.numel() for m in msgs)

        def enc_all():
            for st, m in zip(state, msgs):
                encode_segment(st["wq"][0], st["wq"][1], st["g"].numel, wspec, out=m)

        wire = {"messages": len(msgs), "message_bytes": mbytes}
        gk = capture(enc_all)
        gk.replay()
        torch.cuda.synchronize(dev)
        evk = time_graph(gk, args.steps)
        torch.cuda.synchronize(dev)
        tk = sum(a.elapsed_time(b) for a, b in evk) / args.steps
        wire["encode"] = {"ms_per_pass": round(tk, 4), "gbs": round(2 * mbytes / (tk * 1e-3) / 1e9, 1),
                          "bytes_per_pass": 2 * mbytes}
        for m in msgs:  # warm the decode path (module load, allocator)
            decode_segment(m)
        torch.cuda.synchronize(dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        flush.fill_(7)
        a.record(stream)
        for m in msgs:  # decode = header parse (14-byte D2H) + one kernel + error check per message
            decode_segment(m)
        b.record(stream)
        torch.cuda.synchronize(dev)
        td = a.elapsed_time(b)
        wire["decode_incl_host_checks"] = {"ms_per_pass": round(td, 4), "gbs": round(2 * mbytes / (td * 1e-3) / 1e9, 1)}
        # the decode kernel alone (headers parsed once; the per-message host checks excluded)
        from paper_2302_02390_b200.wire import decode_kernels
        dk = decode_kernels(msgs)
        gk = capture(dk)
        gk.replay()
        torch.cuda.synchronize(dev)
        evk = time_graph(gk, args.steps)
        torch.cuda.synchronize(dev)
        tk = sum(a.elapsed_time(b) for a, b in evk) / args.steps
        wire["decode"] = {"ms_per_pass": round(tk, 4), "gbs": round(2 * mbytes / (tk * 1e-3) / 1e9, 1),
                          "bytes_per_pass": 2 * mbytes}

    # ---- K4 with the fused lattice-projected step (world 1) ----
    lattice = None
    if world == 1 and not args.no_levels:
        from paper_2302_02390_b200.lattice import LatticeStep, dequant_accumulate_lattice, shift_key
        for gi, st in enumerate(state):
            quantize_segments([(st["grad"], 0, SegmentKey(0, 0, gi, 2, 0))], gspec, out=[st["gq"]])
            st["x"] = torch.randn(st["g"].numel, generator=gen, device=dev).mul_(0.02)
        lsteps = [LatticeStep(0.25, 1e-4, shift_key(0, 0, gi)) for gi in range(len(state))]

        def lat_all():
            for st, ls in zip(state, lsteps):
                dequant_accumulate_lattice([st["gq"]], st["g"].numel, gspec, 1, st["x"], ls)

        lb = sum(codes_bytes(st["g"].numel, gspec) + 12 * num_buckets(st["g"].numel, args.bucket)
                 + 8 * st["g"].numel for st in state)  # codes + meta in, fp32 iterate read + written
        gk = capture(lat_all)
        gk.replay()
        torch.cuda.synchronize(dev)
        evk = time_graph(gk, args.steps)
        torch.cuda.synchronize(dev)
        tk = sum(a.elapsed_time(b) for a, b in evk) / args.steps
        lattice = {"K4_lattice_step": {"ms_per_pass": round(tk, 4), "gbs": round(lb / (tk * 1e-3) / 1e9, 1),
                                       "frac_of_hbm_peak": round(lb / (tk * 1e-3) / 1e9 / hbm_peak, 4),
                                       "bytes_per_pass": lb, "x_dtype": "f32", "launches_per_pass": len(state)}}

    # ---- e2e: through the C-ABI communicator, host buffers, copies inside the timed region ----
    e2e = None
    if not args.no_e2e:
        # Pinned host inputs (each group's shard and gradient) and results.  Inside one
        # step the copies overlap the collectives and each other: shards H2D in forward
        # order and gradients in backward order on a copy stream; each collective waits
        # only for its own input; each reduced shard goes D2H on a second copy stream
        # as soon as its RS finishes (full-duplex PCIe; nothing crosses steps).
        host = []
        for st in state:
            host.append(dict(shard=st["shard"].cpu().pin_memory(), grad=st["grad"].cpu().pin_memory(),
                             res=torch.empty(max(st["n"], 1), dtype=torch.float32).pin_memory()))
        bi = sum(h["shard"].numel() * 4 + h["grad"].numel() * 4 for h in host)
        bo = sum(st["n"] * 4 for st in state)
        h2d, d2h = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        comm.set_sm_budget(0)  # the e2e step is PCIe-bound: full-GPU collectives
        rs_comm.set_sm_budget(0)
        # The last gradient of the backward order streams through in bucket-aligned chunks
        # (H2D -> RS -> D2H per chunk), so its result copy does not wait for the whole gradient:
        # only the final chunk's D2H is left after the last H2D byte.  Same codes and results
        # (comm.split_segments).
        from paper_2302_02390_b200.comm import split_segments
        e2e_chunk = 16 << 20  # bytes of gradient per chunk
        for gi, st in enumerate(state):  # only the last gradient of the backward order is chunked
            nch = max(1, -(-st["g"].numel * 4 // e2e_chunk)) if gi == 0 else 1
            st["gparts"] = split_segments(st["segs"], args.bucket, nch)

        def step_e2e():
            main = torch.cuda.current_stream(dev)
            fork = torch.cuda.Event()
            fork.record(main)
            h2d.wait_event(fork)
            d2h.wait_event(fork)
            ev_shard, ev_grad = [], {}
            with torch.cuda.stream(h2d):
                for st, h in zip(state, host):
                    st["shard"].copy_(h["shard"], non_blocking=True)
                    e = torch.cuda.Event()
                    e.record(h2d)
                    ev_shard.append(e)
                for gi in range(len(state) - 1, -1, -1):
                    st, base = state[gi], state[gi]["segs"][0][0]
                    ev_grad[gi] = []
                    for sub in st["gparts"]:
                        for s0, n0 in sub:
                            if n0:
                                st["grad"][s0 - base: s0 - base + n0].copy_(
                                    host[gi]["grad"][s0 - base: s0 - base + n0], non_blocking=True)
                        e = torch.cuda.Event()
                        e.record(h2d)
                        ev_grad[gi].append(e)
            for gi, st in enumerate(state):
                main.wait_event(ev_shard[gi])
                comm.all_gather(st["shard"], st["segs"], SegmentKey(0, 0, gi, 0, 0), st["full"])
            rs_s = main if args.serial else rs_stream
            for gi in range(len(state) - 1, -1, -1):
                st, h = state[gi], host[gi]
                comm.all_gather(st["shard"], st["segs"], SegmentKey(0, 0, gi, 1, 0), st["full"])
                e = torch.cuda.Event()
                e.record(main)
                rs_s.wait_event(e)
                base, s_me = st["segs"][0][0], st["segs"][rank][0]
                for sub, eg in zip(st["gparts"], ev_grad[gi]):
                    rs_s.wait_event(eg)
                    o0, on = sub[rank][0] - s_me, sub[rank][1]
                    with torch.cuda.stream(rs_s):
                        rs_comm.reduce_scatter(st["grad"][sub[0][0] - base:], sub, SegmentKey(0, 0, gi, 2, rank),
                                               st["gshard"][o0:])
                        done = torch.cuda.Event()
                        done.record(rs_s)
                    if on:
                        d2h.wait_event(done)
                        with torch.cuda.stream(d2h):
                            h["res"][o0: o0 + on].copy_(st["gshard"][o0: o0 + on], non_blocking=True)
            for sidestream in (rs_stream, h2d, d2h):
                main.wait_stream(sidestream)
            advance_counter(step_ctr)

        step_e2e()
        torch.cuda.synchronize(dev)
        if args.check_e2e:  # the chunked e2e results == one unchunked RS per group at the same step word
            advance_counter(step_ctr, -1)
            for gi, (st, h) in enumerate(zip(state, host)):
                ref = torch.empty_like(st["gshard"])
                rs_comm.reduce_scatter(st["grad"], st["segs"], SegmentKey(0, 0, gi, 2, rank), ref)
                torch.cuda.synchronize(dev)
                if not torch.equal(ref[: st["n"]].cpu(), h["res"][: st["n"]]):
                    raise SystemExit(f"e2e check failed for group {gi}")
            advance_counter(step_ctr, 1)
            print(f"[rank {rank}] e2e chunked results match the unchunked reduce-scatter", file=sys.stderr)
        barrier()
        g_e2e = capture(step_e2e)
        g_e2e.replay()
        barrier()
        ev = time_graph(g_e2e, args.steps)
        barrier()
        ems = sum(a.elapsed_time(b) for a, b in ev)
        if world > 1:
            t = torch.tensor([ems], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": round(world * 12.0 * N_total / (ems / args.steps * 1e-3) / 1e9, 2), "unit": "GB/s",
               "h2d_bytes_per_step": bi, "d2h_bytes_per_step": bo, "ms_per_step": round(ems / args.steps, 3),
               "path": "QSDPComm -> qsdp_all_gather / qsdp_reduce_scatter (C ABI), pinned host buffers; "
                       "per-group H2D / D2H copies on two copy streams overlapping the collectives inside "
                       "the step (the last gradient in 16 MB bucket-aligned chunks: H2D -> RS -> D2H); one CUDA "
                       "graph per step"}

    # ---- GPT step/s: FSDP2 training step, unquantized (fp32 NCCL) vs QSDP comms ----
    gpt = None
    if not args.no_gpt and world == 1:
        gpt = {"skipped": "world 1: FSDP2 issues no collectives (QSDP and fp32 FSDP are the same step); "
                          "measured at --gpus N > 1"}
    elif not args.no_gpt:
        try:
            from paper_2302_02390_b200.gpt_train import build_model, run_training, shard_model
            gpt = {"model": args.model, "batch_per_gpu": args.gpt_batch, "seq": args.gpt_seq,
                   "data": "synthetic tokens", "timing": "CUDA events per step, max over ranks"}
            for mode in ("fsdp", "qsdp"):
                model = build_model(args.model, dev, seed=0)
                ctx = shard_model(model, mode, wspec, gspec)
                _, times = run_training(model, ctx, steps=args.gpt_steps, batch=args.gpt_batch, seq=args.gpt_seq,
                                        warmup=2)
                times = sorted(times)
                med = times[len(times) // 2]
                gpt[mode] = {"ms_per_step": round(med, 2), "steps_per_s": round(1e3 / med, 3)}
                if ctx is not None:
                    ctx.close()
                del model
                torch.cuda.empty_cache()
            gpt["qsdp_speedup"] = round(gpt["fsdp"]["ms_per_step"] / gpt["qsdp"]["ms_per_step"], 3)
            if world == 1:
                gpt["note"] = "world 1: FSDP2 issues no collectives, both modes are identical"
        except Exception as e:  # the GB/s metric stands on its own
            gpt = {"error": f"{type(e).__name__}: {e}"[:300]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = run_cpu_baseline(args, world)

    if rank == 0:
        line = {
            "metric": "quantized all-gather+reduce-scatter effective GB/s", "value": round(value, 2),
            "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": dict(bench_config(args, world, len(groups), N_total), **{
                "l2": "256 MB L2 flush between timed steps (outside the events: the step then pays the "
                      "write-back of the flush's dirty lines in place of its own trailing ones); per-step "
                      "working set 3 GB > 126 MB L2",
                "execution": "one CUDA graph per step (device step counter), "
                             + ("quantize + barrier + dequantize launches per collective" if world > 1
                                else "one quantizer launch (fused dequant) per collective")
                             + f"; {K} collectives of each kind in flight (FSDP2 prefetch depth; streams + "
                               "communicators per kind), RS(i) after AG_bwd(i)"}),
            "roofline": roofline, "kernels": kernels, "kernels_unfused": kernels_unfused if world == 1 else None, "cpu_baseline": cpu, "e2e": e2e, "gpt": gpt,
            "levels": levels, "philox": philox, "wire": wire, "lattice": lattice,
            "gpu_launches": n_launch * args.steps, "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    for c in set(ag_comms + rs_comms):
        c.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
