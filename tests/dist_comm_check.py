"""Multi-GPU check of QSDPComm (C1/C2 over NVLink peer memory); run with
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tests/dist_comm_check.py
Every rank checks its all-gather output and its reduce-scatter shard bit-exactly
against the oracle's single-process protocol (sharded.py:323-433)."""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import oracle as O  # noqa: E402  (checker only)
from paper_2302_02390_b200.comm import QSDPComm, plan_segments  # noqa: E402
from paper_2302_02390_b200.quantize import QuantSpec, SegmentKey  # noqa: E402


def main():
    dist.init_process_group("nccl")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    failures = 0
    cases = [(1 << 20, 1024, 8, 8, 1, True), (3 * 1024 * 1024 + 777, 1024, 8, 4, 1, True),
             (1 << 22, 1024, 8, 8, 1024, True), (1 << 22, 1024, 8, 8, 1024, False), (50000, 64, 6, 4, 1, True),
             (200000, 256, 4, 2, 256, True), (200000, 512, 16, 8, 1, False)]
    for size, bucket, wb, gb, pad, fused in cases:
        segs = plan_segments(size, world, pad)
        maxseg = max(n for _, n in segs)
        comm = QSDPComm(maxseg, QuantSpec(wb, bucket, "shift"), QuantSpec(gb, bucket, "uniform_stochastic"))
        comm.set_fused(fused)
        rng = np.random.default_rng(size)
        full = (rng.standard_normal(size) * 0.02).astype(np.float32)
        grads = [(np.random.default_rng(size + 1 + p).standard_normal(size) * 1e-3).astype(np.float32)
                 for p in range(world)]
        for step in range(3):
            s, n = segs[rank]
            shard = torch.from_numpy(full[s:s + n]).to(dev)
            out = torch.empty(size, dtype=torch.float32, device=dev)
            comm.all_gather(shard, segs, SegmentKey(0, step, 4, step % 2, 0), out)
            exp = np.zeros(size)
            for q, (sq, nq) in enumerate(segs):
                if nq:
                    c, m, _ = O.quantize_segment(full[sq:sq + nq], sq, bucket, wb, 0, (0, step, 4, step % 2, 0), 8)
                    exp[sq:sq + nq] = O.dequantize_segment(c, m, nq, bucket, wb, 8)
            ok_ag = np.array_equal(out.cpu().numpy(), exp.astype(np.float32))
            g = torch.from_numpy(grads[rank]).to(dev)
            sh = torch.empty(max(n, 1), dtype=torch.float32, device=dev)
            comm.reduce_scatter(g, segs, SegmentKey(0, step, 4, 2, rank), sh)
            acc = np.zeros(n)
            for p in range(world):
                if n:
                    c, m, _ = O.quantize_segment(grads[p][s:s + n], s, bucket, gb, 1, (0, step, 4, 2, p), 8)
                    acc = acc + O.dequantize_segment(c, m, n, bucket, gb, 8)
            ok_rs = np.array_equal(sh[:n].cpu().numpy(), (acc / world).astype(np.float32))
            if not (ok_ag and ok_rs):
                failures += 1
                print(f"rank {rank} size {size} fused {fused} step {step}: ag {ok_ag} rs {ok_rs}", flush=True)
        # graph capture of one AG + RS with the step read on the device (epoch on device too)
        from paper_2302_02390_b200.quantize import advance_counter
        ctr = torch.zeros(1, dtype=torch.int64, device=dev)
        comm.set_step_source(ctr)
        s, n = segs[rank]
        shard = torch.from_numpy(full[s:s + n]).to(dev)
        out = torch.empty(size, dtype=torch.float32, device=dev)
        g = torch.from_numpy(grads[rank]).to(dev)
        sh = torch.empty(max(n, 1), dtype=torch.float32, device=dev)

        def step():
            comm.all_gather(shard, segs, SegmentKey(0, 100, 4, 0, 0), out)
            comm.reduce_scatter(g, segs, SegmentKey(0, 100, 4, 2, rank), sh)
            advance_counter(ctr)
        step()
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        for rep in range(3):
            stepno = int(ctr.item())
            graph.replay()
            torch.cuda.synchronize()
            exp = np.zeros(size)
            for q, (sq, nq) in enumerate(segs):
                if nq:
                    c, m, _ = O.quantize_segment(full[sq:sq + nq], sq, bucket, wb, 0, (0, 100 + stepno, 4, 0, 0), 8)
                    exp[sq:sq + nq] = O.dequantize_segment(c, m, nq, bucket, wb, 8)
            acc = np.zeros(n)
            for p in range(world):
                if n:
                    c, m, _ = O.quantize_segment(grads[p][s:s + n], s, bucket, gb, 1, (0, 100 + stepno, 4, 2, p), 8)
                    acc = acc + O.dequantize_segment(c, m, n, bucket, gb, 8)
            ok = np.array_equal(out.cpu().numpy(), exp.astype(np.float32)) and \
                np.array_equal(sh[:n].cpu().numpy(), (acc / world).astype(np.float32))
            if not ok:
                failures += 1
                print(f"rank {rank} size {size} graph replay {rep}: mismatch", flush=True)
        comm.close()
    failures += levels_all_gather(rank, world, dev)
    failures += lattice_reduce_scatter(rank, world, dev)
    failures += pipelined(rank, world, dev)
    t = torch.tensor([failures], device=dev)
    dist.all_reduce(t)
    if rank == 0:
        print(f"dist_comm_check world={world}: {'OK' if t.item() == 0 else 'FAILED'}", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if t.item() == 0 else 1)


def levels_all_gather(rank, world, dev):
    """C1 with learned weight levels vs the oracle's levels codec."""
    from paper_2302_02390_b200.levels import LevelTable
    fails = 0
    for size, bucket, wb in [(1 << 20, 1024, 5), (300001, 256, 6)]:
        segs = plan_segments(size, world, 1)
        g = np.random.default_rng(3).standard_normal(50000)
        q = O.learn_levels((g - g.min()) / (g.max() - g.min()), np.linspace(0.0, 1.0, 1 << wb), 0.01)
        comm = QSDPComm(max(n for _, n in segs), QuantSpec(wb, bucket, "levels"), QuantSpec(8, bucket, "uniform_stochastic"),
                        weight_levels=LevelTable(q))
        full = (np.random.default_rng(size).standard_normal(size) * 0.02).astype(np.float32)
        s, n = segs[rank]
        out = torch.empty(size, dtype=torch.float32, device=dev)
        for step in range(2):
            comm.all_gather(torch.from_numpy(full[s:s + n]).to(dev), segs, SegmentKey(0, step, 1, 0, 0), out)
            exp = np.zeros(size)
            for sq, nq in segs:
                if nq:
                    c, m, _ = O.quantize_levels_segment(full[sq:sq + nq], bucket, wb, q)
                    exp[sq:sq + nq] = O.dequantize_levels_segment(c, m, nq, bucket, wb, q)
            if not np.array_equal(out.cpu().numpy(), exp.astype(np.float32)):
                fails += 1
                print(f"rank {rank} levels size {size} step {step}: mismatch", flush=True)
        comm.close()
    return fails


def lattice_reduce_scatter(rank, world, dev):
    """C2 + the fused lattice step on every owner's shard vs the oracle."""
    from paper_2302_02390_b200.lattice import LatticeStep, shift_key
    fails = 0
    size, bucket, gb, d, cc = 700001, 1024, 8, 2e-4, 0.3
    segs = plan_segments(size, world, bucket)
    comm = QSDPComm(max(n for _, n in segs), QuantSpec(8, bucket, "shift"), QuantSpec(gb, bucket, "uniform_stochastic"))
    grads = [(np.random.default_rng(50 + p).standard_normal(size) * 1e-3).astype(np.float32) for p in range(world)]
    x_full = np.random.default_rng(99).standard_normal(size)
    s, n = segs[rank]
    x = torch.from_numpy(x_full[s:s + n].copy()).to(dev)
    for step in range(2):
        comm.reduce_scatter_lattice(torch.from_numpy(grads[rank]).to(dev), segs, SegmentKey(0, step, 6, 2, rank), x,
                                    LatticeStep(cc, d, shift_key(0, step, 6)))
        acc = np.zeros(n)
        for p in range(world):
            c, m, _ = O.quantize_segment(grads[p][s:s + n], s, bucket, gb, 1, (0, step, 6, 2, p), 8)
            acc = acc + O.dequantize_segment(c, m, n, bucket, gb, 8)
        r = -d / 2 + d * O.PCG64(0, step, 6, 3, 0, 0).random()
        x_full[s:s + n] = d * np.round((x_full[s:s + n] - cc * (acc / world) - r) / d) + r
        if not np.array_equal(x.cpu().numpy(), x_full[s:s + n]):
            fails += 1
            print(f"rank {rank} lattice step {step}: mismatch", flush=True)
    comm.close()
    return fails


def pipelined(rank, world, dev):
    """PipelinedComm (bucket-aligned sub-collectives on two comms / streams) equals one QSDPComm call."""
    from paper_2302_02390_b200.comm import PipelinedComm
    fails = 0
    for size, bucket, chunks in [(3 * 1024 * 1024 + 5, 1024, 4), (200003, 256, 3)]:
        segs = plan_segments(size, world, bucket)
        ms = max(n for _, n in segs)
        ws, gs = QuantSpec(8, bucket, "shift"), QuantSpec(4, bucket, "uniform_stochastic")
        one, pipe = QSDPComm(ms, ws, gs), PipelinedComm(ms, ws, gs, chunks=chunks)
        full = torch.randn(size, device=dev) * 0.02
        g = torch.randn(size, device=dev) * 1e-3
        s, n = segs[rank]
        a, b = torch.empty(size, device=dev), torch.empty(size, device=dev)
        one.all_gather(full[s:s + n], segs, SegmentKey(1, 2, 3, 0, 0), a)
        pipe.all_gather(full[s:s + n], segs, SegmentKey(1, 2, 3, 0, 0), b)
        ra, rb = torch.empty(max(n, 1), device=dev), torch.empty(max(n, 1), device=dev)
        one.reduce_scatter(g, segs, SegmentKey(1, 2, 3, 2, rank), ra)
        pipe.reduce_scatter(g, segs, SegmentKey(1, 2, 3, 2, rank), rb)
        torch.cuda.synchronize()
        if not (torch.equal(a, b) and torch.equal(ra[:n], rb[:n])):
            fails += 1
            print(f"rank {rank} pipelined size {size}: mismatch", flush=True)
        one.close()
        pipe.close()
    return fails


if __name__ == "__main__":
    main()
