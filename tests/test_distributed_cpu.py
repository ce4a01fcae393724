"""CPU, world_size 2 over gloo: the multi-rank host logic of C1/C2.

Each rank follows the product's schedule (comm.all_gather_plan /
reduce_scatter_plan), with the oracle standing in for the kernels (tests only)
and gloo standing in for NVLink; the result must equal the single-process
protocol (sharded.py:323-433) bit-for-bit, and the per-rank sent bits must sum
to the reference ledger's totals."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2302_02390_b200.comm import all_gather_plan, plan_segments, reduce_scatter_plan, sent_bits
from paper_2302_02390_b200.quantize import QuantSpec, SegmentKey

WORLD = 2
SIZE = 5000 + 3  # ragged: remainder on the last rank


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import oracle as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        rng = np.random.default_rng(0)
        full = rng.standard_normal(SIZE) * 0.02
        grads = [np.random.default_rng(1 + p).standard_normal(SIZE) * 1e-3 for p in range(WORLD)]
        segs = plan_segments(SIZE, WORLD)
        bucket, wb, gb = 256, 8, 4
        # ---- all-gather ----
        quant, pull = all_gather_plan(rank, WORLD, segs, SegmentKey(7, 3, 5, 1, 99))
        (s, n, k), = quant
        codes, meta, _ = O.quantize_segment(full[s:s + n], s, bucket, wb, 0,
                                            (k.root_seed, k.step, k.layer, k.phase, k.worker))
        slots = [None] * WORLD
        dist.all_gather_object(slots, (codes, meta))
        out = np.zeros(SIZE)
        for p, off, ln in pull:
            out[off:off + ln] = O.dequantize_segment(slots[p][0], slots[p][1], ln, bucket, wb)
        ref = O.gather(full, WORLD, bucket, wb, 7, 3, 5, 1)
        ok_ag = np.array_equal(out, ref)
        # ---- reduce-scatter ----
        quant, pull = reduce_scatter_plan(rank, WORLD, segs, SegmentKey(7, 3, 5, 2, 0))
        mine = {}
        for dst, s2, n2, k2 in quant:
            mine[dst] = O.quantize_segment(grads[rank][s2:s2 + n2], s2, bucket, gb, 1,
                                           (k2.root_seed, k2.step, k2.layer, k2.phase, k2.worker))[:2]
        allq = [None] * WORLD
        dist.all_gather_object(allq, mine)
        s, n = segs[rank]
        acc = np.zeros(n)
        for p in pull:
            c, m = allq[p][rank]
            acc = acc + O.dequantize_segment(c, m, n, bucket, gb)
        ok_rs = np.array_equal(acc / WORLD, O.reduce_scatter(grads, bucket, gb, 7, 3, 5)[rank])
        bits = (sent_bits("allgather", rank, WORLD, segs, QuantSpec(wb, bucket, "shift")),
                sent_bits("reducescatter", rank, WORLD, segs, QuantSpec(gb, bucket, "uniform_stochastic")))
        q.put((rank, ok_ag, ok_rs, bits))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_protocol_over_gloo(oracle):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(WORLD)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_ag, ok_rs, _ in res:
        assert ok_ag, f"rank {rank} all-gather differs from the single-process protocol"
        assert ok_rs, f"rank {rank} reduce-scatter differs from the single-process protocol"
    # ledger: per-rank sends sum to the reference's totals
    segs = plan_segments(SIZE, WORLD)
    ag = sum(r[3][0] for r in res)
    rs = sum(r[3][1] for r in res)
    exp_ag = sum(oracle.message_size_bits(n, 256, 8) * (WORLD - 1) for _, n in segs)
    exp_rs = sum(oracle.message_size_bits(n, 256, 4) for q_, (_, n) in enumerate(segs) for p in range(WORLD)
                 if p != q_)
    assert (ag, rs) == (exp_ag, exp_rs)


def test_plans_cover_every_rank():
    segs = plan_segments(10, 4, pad_to=4)
    for r in range(4):
        q, pull = all_gather_plan(r, 4, segs, SegmentKey(0, 1, 2, 0, 5))
        assert all(k.worker == 0 for *_, k in q)
        assert [p for p, _, _ in pull] == [0, 1, 2]  # rank 3's segment is empty
        q, pull = reduce_scatter_plan(r, 4, segs, SegmentKey(0, 1, 2, 2, 0))
        assert all(k.worker == r for *_, k in q)
        assert pull == ([0, 1, 2, 3] if segs[r][1] else [])
