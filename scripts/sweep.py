"""Standalone C1 / C2 sweep: fp32 tensors of 1 MB .. 1 GB
(N = 2^18 .. 2^28), w/g widths 8 and 4, bucket 1024, one process per GPU.

Each point is 10 back-to-back calls of one collective captured in a CUDA graph,
timed with CUDA events after an L2 flush, max over ranks.  Reported per point:
effective GB/s = 4N / T (the nccl-tests algbw convention on the fp32 tensor), bus
GB/s = c N (P-1)/P / T against 900 GB/s per direction, the fraction of the roofline
T* = max(HBM bytes / peak, NVLink bytes / 900 GB/s) (HBM peak from MEASURED_PEAKS.json)
with the per-element bytes of §8(d), and -- counter evidence -- the NVLink data
bytes rank 0's GPU transmitted during the timed replays (nvidia-smi nvlink -gt d,
read before / after) per collective, next to the algorithmic c N (P-1)/P:

    C1 all-gather       HBM 4/P + o + 2c     NVLink c (P-1)/P
    C2 reduce-scatter   HBM 4 + 2c + 4/P     NVLink c (P-1)/P      (c = b/8 + 12/S, o = 4)

    python -m torch.distributed.run --nproc-per-node P --master-addr 127.0.0.1 scripts/sweep.py > sweep_pP.jsonl
"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_02390_b200.comm import PipelinedComm, QSDPComm, plan_segments  # noqa: E402
from paper_2302_02390_b200.quantize import QuantSpec, SegmentKey, advance_counter  # noqa: E402

NVL = 900e9
try:
    HBM = float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                            "MEASURED_PEAKS.json")))["hbm_gbs"]) * 1e9
except Exception:
    HBM = 6555.2e9  # B200_PROFILING.md fallback


def nvlink_tx_bytes(index: int):
    """Data bytes this GPU has transmitted over all its NVLinks (nvidia-smi nvlink -gt d), or None."""
    import re
    import subprocess
    try:
        out = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", str(index)], capture_output=True,
                             text=True, timeout=30).stdout
    except Exception:
        return None
    tx = [int(m) for m in re.findall(r"Data Tx:\s*(\d+)\s*KiB", out)]
    return sum(tx) * 1024 if tx else None


def main():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    S = 1024
    flush = torch.empty(64 << 20, dtype=torch.int32, device=dev)
    ctr = torch.zeros(1, dtype=torch.int64, device=dev)
    for logn in [int(v) for v in os.environ.get("SWEEP_LOGN", "18,20,22,24,26,28").split(",")]:
        n = 1 << logn
        segs = plan_segments(n, world, S)
        s0, ns = segs[rank]
        x = torch.randn(ns, device=dev) * 0.02
        g = torch.randn(n, device=dev) * 1e-3
        full = torch.empty(n, device=dev)
        shard = torch.empty(max(ns, 1), device=dev)
        for bits in [int(v) for v in os.environ.get("SWEEP_BITS", "8,4").split(",")]:
            pipe = int(os.environ.get("PIPE", "0"))  # >1: PipelinedComm with this many chunks
            ctor = (lambda *a, **k: PipelinedComm(*a, chunks=pipe, **k)) if pipe > 1 else QSDPComm
            comm = ctor(max(m for _, m in segs), QuantSpec(bits, S, "shift"), QuantSpec(bits, S, "uniform_stochastic"),
                        device=dev)
            comm.set_step_source(ctr)
            c = bits / 8 + 12 / S
            for kind in ("allgather", "reducescatter"):
                def one():
                    for i in range(10):
                        if kind == "allgather":
                            comm.all_gather(x, segs, SegmentKey(0, 0, i, 0, 0), full)
                        else:
                            comm.reduce_scatter(g, segs, SegmentKey(0, 0, i, 2, rank), shard)
                    advance_counter(ctr)
                one()
                torch.cuda.synchronize()
                gr = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gr):
                    one()
                gr.replay()
                torch.cuda.synchronize()
                tot = 0.0
                reps = 5
                tx0 = nvlink_tx_bytes(local) if (rank == 0 and world > 1) else None
                for r in range(reps):
                    flush.fill_(r)
                    if world > 1:
                        dist.barrier()
                    torch.cuda.synchronize()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    gr.replay()
                    b.record()
                    torch.cuda.synchronize()
                    tot += a.elapsed_time(b)
                tx1 = nvlink_tx_bytes(local) if tx0 is not None else None
                t = torch.tensor([tot / reps / 10 * 1e-3], device=dev, dtype=torch.float64)  # s per collective
                if world > 1:
                    dist.all_reduce(t, op=dist.ReduceOp.MAX)
                T = float(t.item())
                P = world
                hbm = (4 / P + 4 + 2 * c) if kind == "allgather" else (4 + 2 * c + 4 / P)
                nvl = c * (P - 1) / P
                tstar = max(hbm * n / HBM, nvl * n / NVL)
                if rank == 0:
                    line = {"P": P, "pipe": pipe, "n": n, "mb_fp32": n * 4 / 2 ** 20, "bits": bits, "collective": kind,
                            "us": round(T * 1e6, 2), "eff_gbs": round(4 * n / T / 1e9, 1),
                            "bus_gbs": round(nvl * n / T / 1e9, 1), "bus_frac_of_900": round(nvl * n / T / NVL, 3),
                            "roofline_eff_gbs": round(4 * n / tstar / 1e9, 1),
                            "frac_of_roofline": round(tstar / T, 3), "hbm_peak_gbs": round(HBM / 1e9, 1)}
                    if tx1 is not None:
                        per = (tx1 - tx0) / (reps * 10)
                        line["nvlink_tx_bytes_per_collective"] = int(per)
                        line["nvlink_tx_algorithmic_bytes"] = int(nvl * n)
                    print(json.dumps(line), flush=True)
            comm.close()
        del x, g, full, shard
        torch.cuda.empty_cache()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
