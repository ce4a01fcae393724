"""Multi-process check of QSDPComm (C1/C2 over peer memory); run with
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tests/dist_comm_check.py
Every rank checks its all-gather output and its reduce-scatter shard bit-exactly
against the oracle's single-process protocol (sharded.py:323-433).

QSDP_SAME_GPU=1 runs every rank on cuda:0 (gloo for the host plumbing: NCCL refuses
two ranks on one device; QSDPComm only needs all_gather_object + barrier for the IPC
handle exchange).  The data path is unchanged -- CUDA IPC mappings of the other
processes' workspaces, the push mirror, the system-scope flag barrier, parity-slot
reuse and the world>1 own-shard fused dequant -- so a one-GPU box exercises the
whole multi-process protocol; only the links are HBM instead of NVLink."""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import oracle as O  # noqa: E402  (checker only)
from paper_2302_02390_b200.comm import QSDPComm, plan_segments  # noqa: E402
from paper_2302_02390_b200.quantize import QuantSpec, SegmentKey  # noqa: E402

SAME_GPU = os.environ.get("QSDP_SAME_GPU", "0") == "1"


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", 0 if SAME_GPU else local)
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo" if SAME_GPU else "nccl")
    rank, world = dist.get_rank(), dist.get_world_size()
    failures = 0
    # (size, bucket, w bits, g bits, pad): pad 1 = shard_bounds, whose rank offsets are
    # not multiples of 4 for the odd sizes (the own-shard fused dequant must then
    # leave that shard to K3's scalar stores -- ADVICE r1)
    # the last three are small collectives (a few buckets per rank, partial last buckets)
    cases = [(1 << 20, 1024, 8, 8, 1), (3 * 1024 * 1024 + 777, 1024, 8, 4, 1), (1000003, 1024, 8, 8, 1),
             (1 << 22, 1024, 8, 8, 1024), (50000, 64, 6, 4, 1),
             (200000, 256, 4, 2, 256), (200000, 512, 16, 8, 1),
             (4003, 1024, 8, 8, 1), (30011, 256, 4, 2, 1), (9000, 512, 16, 8, 1)]
    for size, bucket, wb, gb, pad in cases:
        segs = plan_segments(size, world, pad)
        maxseg = max(n for _, n in segs)
        comm = QSDPComm(maxseg, QuantSpec(wb, bucket, "shift"), QuantSpec(gb, bucket, "uniform_stochastic"))
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
                print(f"rank {rank} size {size} step {step}: ag {ok_ag} rs {ok_rs}", flush=True)
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
    failures += offset_views(rank, world, dev)
    failures += philox_collectives(rank, world, dev)
    failures += group_pieces(rank, world, dev)
    failures += levels_all_gather(rank, world, dev)
    failures += lattice_reduce_scatter(rank, world, dev)
    failures += pipelined(rank, world, dev)
    failures += missed_barrier(rank, world, dev)
    t = torch.tensor([failures], device="cpu" if SAME_GPU else dev)
    dist.all_reduce(t)
    if rank == 0:
        print(f"dist_comm_check world={world}{' (all ranks on cuda:0)' if SAME_GPU else ''}: "
              f"{'OK' if t.item() == 0 else 'FAILED'}", flush=True)
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


def offset_views(rank, world, dev):
    """Outputs that are offset views (out[1:], shard[3:]) of larger buffers: no
    alignment is assumed anywhere on the path."""
    fails = 0
    size, bucket = 777777, 1024
    segs = plan_segments(size, world, 1)
    comm = QSDPComm(max(n for _, n in segs), QuantSpec(8, bucket, "shift"), QuantSpec(8, bucket, "uniform_stochastic"))
    full = (np.random.default_rng(7).standard_normal(size) * 0.02).astype(np.float32)
    grads = [(np.random.default_rng(70 + p).standard_normal(size) * 1e-3).astype(np.float32) for p in range(world)]
    s, n = segs[rank]
    for step in range(2):
        out_big = torch.full((size + 1,), float("nan"), device=dev)
        comm.all_gather(torch.from_numpy(full[s:s + n]).to(dev), segs, SegmentKey(3, step, 2, 0, 0), out_big[1:])
        exp = np.zeros(size)
        for sq, nq in segs:
            c, m, _ = O.quantize_segment(full[sq:sq + nq], sq, bucket, 8, 0, (3, step, 2, 0, 0), 8)
            exp[sq:sq + nq] = O.dequantize_segment(c, m, nq, bucket, 8, 8)
        ok_ag = np.array_equal(out_big[1:].cpu().numpy(), exp.astype(np.float32))
        g_big = torch.zeros(size + 3, device=dev)
        g_big[3:] = torch.from_numpy(grads[rank]).to(dev)
        sh_big = torch.full((n + 1,), float("nan"), device=dev)
        comm.reduce_scatter(g_big[3:], segs, SegmentKey(3, step, 2, 2, rank), sh_big[1:])
        acc = np.zeros(n)
        for p in range(world):
            c, m, _ = O.quantize_segment(grads[p][s:s + n], s, bucket, 8, 1, (3, step, 2, 2, p), 8)
            acc = acc + O.dequantize_segment(c, m, n, bucket, 8, 8)
        ok_rs = np.array_equal(sh_big[1:].cpu().numpy(), (acc / world).astype(np.float32))
        if not (ok_ag and ok_rs):
            fails += 1
            print(f"rank {rank} offset views step {step}: ag {ok_ag} rs {ok_rs}", flush=True)
    comm.close()
    return fails


def missed_barrier(rank, world, dev):
    """Failure detection: rank world-1 skips a collective; the others' barrier gives up
    after the timeout and the communicator reports QSDP_EPEER instead of hanging."""
    from paper_2302_02390_b200._lib import QSDPError
    if world < 2:
        return 0
    fails = 0
    size = 100000
    segs = plan_segments(size, world, 1)
    comm = QSDPComm(max(n for _, n in segs), QuantSpec(8, 1024, "shift"), QuantSpec(8, 1024, "uniform_stochastic"))
    comm.set_timeout(1500)
    s, n = segs[rank]
    x = torch.randn(n, device=dev)
    out = torch.empty(size, device=dev)
    if rank != world - 1:
        comm.all_gather(x, segs, SegmentKey(0, 0, 0, 0, 0), out)
        torch.cuda.synchronize()
        try:
            comm.check()
            fails += 1
            print(f"rank {rank}: missed barrier not detected", flush=True)
        except QSDPError as e:
            if "did not arrive" not in str(e):
                fails += 1
                print(f"rank {rank}: unexpected error {e}", flush=True)
        try:  # later collectives fail fast
            comm.all_gather(x, segs, SegmentKey(0, 1, 0, 0, 0), out)
            fails += 1
            print(f"rank {rank}: collective after a failed barrier did not raise", flush=True)
        except QSDPError:
            pass
    dist.barrier()
    comm.close()
    return fails


def philox_collectives(rank, world, dev):
    """C1/C2 with the counter-based noise (QSDP_NOISE_PHILOX4x64) at world > 1 (pull form)."""
    fails = 0
    for size, bucket in ((500009, 1024), (20011, 1024)):  # the second: a small collective
        fails += _philox_case(rank, world, dev, size, bucket)
    return fails


def _philox_case(rank, world, dev, size, bucket):
    fails = 0
    segs = plan_segments(size, world, 1)
    ws, gs = QuantSpec(8, bucket, "shift", "philox"), QuantSpec(4, bucket, "uniform_stochastic", "philox")
    comm = QSDPComm(max(n for _, n in segs), ws, gs)
    full = (np.random.default_rng(17).standard_normal(size) * 0.02).astype(np.float32)
    grads = [(np.random.default_rng(170 + p).standard_normal(size) * 1e-3).astype(np.float32) for p in range(world)]
    s, n = segs[rank]
    for step in range(2):
        out = torch.empty(size, device=dev)
        comm.all_gather(torch.from_numpy(full[s:s + n]).to(dev), segs, SegmentKey(5, step, 1, 0, 0), out)
        exp = np.zeros(size)
        for sq, nq in segs:
            c, m, _ = O.quantize_segment(full[sq:sq + nq], sq, bucket, 8, 0, (5, step, 1, 0, 0), 8, noise=1)
            exp[sq:sq + nq] = O.dequantize_segment(c, m, nq, bucket, 8, 8)
        sh = torch.empty(max(n, 1), device=dev)
        comm.reduce_scatter(torch.from_numpy(grads[rank]).to(dev), segs, SegmentKey(5, step, 1, 2, rank), sh)
        acc = np.zeros(n)
        for p in range(world):
            c, m, _ = O.quantize_segment(grads[p][s:s + n], s, bucket, 4, 1, (5, step, 1, 2, p), 8, noise=1)
            acc = acc + O.dequantize_segment(c, m, n, bucket, 4, 8)
        if not (np.array_equal(out.cpu().numpy(), exp.astype(np.float32))
                and np.array_equal(sh[:n].cpu().numpy(), (acc / world).astype(np.float32))):
            fails += 1
            print(f"rank {rank} philox step {step}: mismatch", flush=True)
    comm.close()
    return fails


def group_pieces(rank, world, dev):
    """qsdp_all_gather_pieces / qsdp_reduce_scatter_pieces: several equal-per-rank pieces at
    fixed offsets of a rank's flat buffer (an FSDP2 group), keyed start = q*stride + offset;
    the gaps between them are full-precision pieces (``raw``: biases / norms, sharded.py:
    359-371, 414-429) carried by the same call -- all-gather: the values cast to the output
    dtype, reduce-scatter: (0.0 + v_0 + ... + v_{P-1}) / P in fp64, rounded once."""
    fails = 0
    rng = np.random.default_rng(23)
    sizes = [5000, 1024 * 7, 333, 4096 * 3 + 8]
    raw_sizes = [5, 3000, 1, 7]  # after each quantized piece
    offs, roffs, off = [], [], 0
    for n, r in zip(sizes, raw_sizes):
        offs.append(off)
        off += n
        roffs.append(off)
        off += r
    for k in range(56):  # 60 full-precision pieces: more than the barrier kernel's table of 48
        raw_sizes.append(1 + k % 5)
        roffs.append(off)
        off += raw_sizes[-1]
    stride = off
    cap = sum(sizes) + len(sizes) * (1024 + 16) + 4 * (sum(raw_sizes) + 4 * len(raw_sizes))
    comm = QSDPComm(cap, QuantSpec(8, 1024, "shift"), QuantSpec(8, 1024, "uniform_stochastic"))
    shards = [[(rng.standard_normal(n) * 0.02).astype(np.float32) for n in sizes] for _ in range(world)]
    rshards = [[(rng.standard_normal(n) * 0.5).astype(np.float32) for n in raw_sizes] for _ in range(world)]
    grads = [(rng.standard_normal(world * stride) * 1e-3).astype(np.float32) for _ in range(world)]
    for out_dt in (torch.float32, torch.bfloat16):
        out = torch.zeros(world * stride, dtype=out_dt, device=dev)
        pieces = [(torch.from_numpy(shards[rank][k]).to(dev), offs[k], sizes[k]) for k in range(len(sizes))]
        pieces += [(torch.from_numpy(rshards[rank][k]).to(dev), roffs[k], raw_sizes[k], True)
                   for k in range(len(raw_sizes))]
        comm.all_gather_pieces(pieces, stride, SegmentKey(2, 3, 4, 1, 0), out)
        got = out.float().cpu().numpy()
        for q in range(world):
            for k, n in enumerate(sizes):
                a = q * stride + offs[k]
                c, m, _ = O.quantize_segment(shards[q][k], a, 1024, 8, 0, (2, 3, 4, 1, 0), 8)
                exp = torch.from_numpy(O.dequantize_segment(c, m, n, 1024, 8, 8).astype(np.float32))
                if not np.array_equal(got[a:a + n], exp.to(out_dt).float().numpy()):
                    fails += 1
                    print(f"rank {rank} pieces AG {out_dt} q {q} k {k}: mismatch", flush=True)
            for k, n in enumerate(raw_sizes):
                a = q * stride + roffs[k]
                exp = torch.from_numpy(rshards[q][k]).to(out_dt).float().numpy()
                if not np.array_equal(got[a:a + n], exp):
                    fails += 1
                    print(f"rank {rank} pieces AG raw {out_dt} q {q} k {k}: mismatch", flush=True)
    rs = torch.zeros(stride, device=dev)
    rs_pieces = list(zip(offs, sizes)) + [(o, n, True) for o, n in zip(roffs, raw_sizes)]
    comm.reduce_scatter_pieces(torch.from_numpy(grads[rank]).to(dev), rs_pieces, stride,
                               SegmentKey(2, 3, 4, 2, rank), rs)
    got = rs.cpu().numpy()
    for k, n in enumerate(sizes):
        a = rank * stride + offs[k]
        acc = np.zeros(n)
        for p in range(world):
            c, m, _ = O.quantize_segment(grads[p][a:a + n], a, 1024, 8, 1, (2, 3, 4, 2, p), 8)
            acc = acc + O.dequantize_segment(c, m, n, 1024, 8, 8)
        if not np.array_equal(got[offs[k]:offs[k] + n], (acc / world).astype(np.float32)):
            fails += 1
            print(f"rank {rank} pieces RS k {k}: mismatch", flush=True)
    for k, n in enumerate(raw_sizes):
        a = rank * stride + roffs[k]
        acc = np.zeros(n)
        for p in range(world):
            acc = acc + grads[p][a:a + n].astype(np.float64)
        if not np.array_equal(got[roffs[k]:roffs[k] + n], (acc / world).astype(np.float32)):
            fails += 1
            print(f"rank {rank} pieces RS raw k {k}: mismatch", flush=True)
    comm.close()
    return fails


if __name__ == "__main__":
    main()
