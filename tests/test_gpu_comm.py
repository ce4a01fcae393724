"""GPU: the C1/C2 communicator.  world=1 in-process; world>1 via torchrun when
the box has several GPUs (tests/dist_comm_check.py)."""

import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from conftest import ROOT
from paper_2302_02390_b200.comm import QSDPComm, plan_segments
from paper_2302_02390_b200.quantize import QuantSpec, SegmentKey

pytestmark = pytest.mark.gpu


def test_single_rank_comm_vs_oracle(oracle):
    dev = torch.device("cuda", 0)
    size = 3 * 1024 * 100 + 11
    comm = QSDPComm(size, QuantSpec(8, 1024, "shift"), QuantSpec(8, 1024, "uniform_stochastic"), device=dev)
    x = (np.random.default_rng(1).standard_normal(size) * 0.02).astype(np.float32)
    xt = torch.from_numpy(x).to(dev)
    for step in range(3):
        out = torch.empty(size, device=dev)
        comm.all_gather(xt, [(0, size)], SegmentKey(0, step, 1, 0, 0), out)
        c, m, _ = oracle.quantize_segment(x, 0, 1024, 8, 0, (0, step, 1, 0, 0), 8)
        exp = oracle.dequantize_segment(c, m, size, 1024, 8, 8).astype(np.float32)
        assert np.array_equal(out.cpu().numpy(), exp)
        sh = torch.empty(size, device=dev)
        comm.reduce_scatter(xt, [(0, size)], SegmentKey(0, step, 1, 2, 0), sh)
        c, m, _ = oracle.quantize_segment(x, 0, 1024, 8, 1, (0, step, 1, 2, 0), 8)
        exp = (np.zeros(size) + oracle.dequantize_segment(c, m, size, 1024, 8, 8)) / 1
        assert np.array_equal(sh.cpu().numpy(), exp.astype(np.float32))
    comm.close()


@pytest.mark.parametrize("ctas,sms", [(1, 0), (1, 37), (0, 20)])
def test_occupancy_caps_keep_results(oracle, ctas, sms):
    """qsdp_comm_set_ctas_per_sm / set_sm_budget size the grids only: same bits as the oracle."""
    dev = torch.device("cuda", 0)
    size = 1024 * 3000 + 77
    comm = QSDPComm(size, QuantSpec(8, 1024, "shift"), QuantSpec(8, 1024, "uniform_stochastic"), device=dev)
    comm.set_ctas_per_sm(ctas)
    comm.set_sm_budget(sms)
    x = (np.random.default_rng(5).standard_normal(size) * 0.02).astype(np.float32)
    xt = torch.from_numpy(x).to(dev)
    out = torch.empty(size, device=dev)
    comm.all_gather(xt, [(0, size)], SegmentKey(3, 1, 2, 0, 0), out)
    c, m, _ = oracle.quantize_segment(x, 0, 1024, 8, 0, (3, 1, 2, 0, 0), 8)
    assert np.array_equal(out.cpu().numpy(), oracle.dequantize_segment(c, m, size, 1024, 8, 8).astype(np.float32))
    sh = torch.empty(size, device=dev)
    comm.reduce_scatter(xt, [(0, size)], SegmentKey(3, 1, 2, 2, 0), sh)
    c, m, _ = oracle.quantize_segment(x, 0, 1024, 8, 1, (3, 1, 2, 2, 0), 8)
    assert np.array_equal(sh.cpu().numpy(), oracle.dequantize_segment(c, m, size, 1024, 8, 8).astype(np.float32))
    comm.close()


def test_graph_replay_with_device_step(oracle):
    """A captured AG+RS replays with the step read on the device (fresh noise per replay)."""
    from paper_2302_02390_b200.quantize import advance_counter
    dev = torch.device("cuda", 0)
    size = 70000
    comm = QSDPComm(size, QuantSpec(8, 1024, "shift"), QuantSpec(4, 1024, "uniform_stochastic"), device=dev)
    ctr = torch.zeros(1, dtype=torch.int64, device=dev)
    comm.set_step_source(ctr)
    x = (np.random.default_rng(3).standard_normal(size) * 0.02).astype(np.float32)
    xt = torch.from_numpy(x).to(dev)
    out = torch.empty(size, device=dev)
    sh = torch.empty(size, device=dev)

    def step():
        comm.all_gather(xt, [(0, size)], SegmentKey(0, 10, 1, 0, 0), out)
        comm.reduce_scatter(xt, [(0, size)], SegmentKey(0, 10, 1, 2, 0), sh)
        advance_counter(ctr)

    step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for rep in range(2):
        stepno = int(ctr.item())
        g.replay()
        torch.cuda.synchronize()
        c, m, _ = oracle.quantize_segment(x, 0, 1024, 8, 0, (0, 10 + stepno, 1, 0, 0), 8)
        assert np.array_equal(out.cpu().numpy(), oracle.dequantize_segment(c, m, size, 1024, 8, 8).astype(np.float32))
        c, m, _ = oracle.quantize_segment(x, 0, 1024, 4, 1, (0, 10 + stepno, 1, 2, 0), 8)
        assert np.array_equal(sh.cpu().numpy(), oracle.dequantize_segment(c, m, size, 1024, 4, 8).astype(np.float32))
    comm.close()


def test_levels_all_gather_single_rank(oracle):
    """C1 with learned weight levels; a missing table fails loudly."""
    from paper_2302_02390_b200.levels import LevelTable
    dev = torch.device("cuda", 0)
    size, bucket, wb = 1024 * 77 + 5, 1024, 6
    q = np.sort(np.random.default_rng(2).uniform(0, 1, 1 << wb))
    comm = QSDPComm(size, QuantSpec(wb, bucket, "levels"), QuantSpec(8, bucket, "uniform_stochastic"), device=dev)
    x = (np.random.default_rng(5).standard_normal(size) * 0.02).astype(np.float32)
    out = torch.empty(size, device=dev)
    with pytest.raises(ValueError, match="LevelTable"):
        comm.all_gather(torch.from_numpy(x).to(dev), [(0, size)], SegmentKey(0, 0, 1, 0, 0), out)
    comm.set_weight_levels(LevelTable(q))
    comm.all_gather(torch.from_numpy(x).to(dev), [(0, size)], SegmentKey(0, 0, 1, 0, 0), out)
    c, m, _ = oracle.quantize_levels_segment(x, bucket, wb, q)
    exp = oracle.dequantize_levels_segment(c, m, size, bucket, wb, q).astype(np.float32)
    assert np.array_equal(out.cpu().numpy(), exp)
    comm.close()


def test_plan_segments():
    assert plan_segments(10, 4) == [(0, 2), (2, 2), (4, 2), (6, 4)]
    assert plan_segments(10, 4, pad_to=4) == [(0, 4), (4, 4), (8, 2), (10, 0)]


def _torchrun(script, nproc, port, extra_env=None, timeout=900):
    env = dict(os.environ, PYTHONPATH=ROOT, **(extra_env or {}))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(ROOT, "tests", script)],
                       capture_output=True, text=True, timeout=timeout, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return r.stdout


@pytest.mark.parametrize("world", [2, 4, 8])
def test_multi_process_comm_one_gpu(world):
    """The one-process-per-rank C1/C2 protocol with every rank on cuda:0 (gloo host
    plumbing): CUDA IPC workspaces of the other processes, the push mirror, the
    flag barrier, parity-slot reuse, the world>1 own-shard fused dequant, graph
    replay, unaligned rank offsets and barrier-timeout failure detection -- bit-exact
    vs the oracle on a one-GPU box (tests/dist_comm_check.py, QSDP_SAME_GPU=1)."""
    out = _torchrun("dist_comm_check.py", world, 29540 + world, {"QSDP_SAME_GPU": "1"})
    assert f"dist_comm_check world={world} (all ranks on cuda:0): OK" in out


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_multi_gpu_comm():
    """One rank per GPU over NVLink, every GPU of the box (up to 8)."""
    n = min(8, torch.cuda.device_count())
    out = _torchrun("dist_comm_check.py", n, 29533)
    assert f"dist_comm_check world={n}: OK" in out


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs (world 1 has no hierarchy)")
def test_hierarchical_comm():
    """Two-level (inter-node / intra-node) C1/C2, every node shape
    dividing the world size, bit-exact vs the oracle (tests/dist_hier_check.py)."""
    n = min(8, torch.cuda.device_count())
    _torchrun("dist_hier_check.py", n, 29534)


def test_group_pieces_world1(oracle):
    """qsdp_all_gather_pieces / qsdp_reduce_scatter_pieces at world 1 (fused epilogue when
    every piece is aligned, K3 otherwise)."""
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(31)
    for sizes, gap in (([4096, 1024 * 3, 700], 0), ([5000, 2048, 129], 3)):
        offs, off = [], 0
        for n in sizes:
            offs.append(off)
            off += n + gap
        comm = QSDPComm(sum(sizes) + len(sizes) * 1040 + 8 * (gap + 4) * len(sizes), QuantSpec(8, 1024, "shift"),
                        QuantSpec(4, 1024, "uniform_stochastic"), device=dev)
        xs = [(rng.standard_normal(n) * 0.02).astype(np.float32) for n in sizes]
        out = torch.zeros(off, device=dev)
        base = torch.from_numpy((rng.standard_normal(off) * 0.3).astype(np.float32)).to(dev)
        raw = [(base[o + n:o + n + gap], o + n, gap, True) for o, n in zip(offs, sizes) if gap]  # full precision
        comm.all_gather_pieces([(torch.from_numpy(x).to(dev), o, n) for x, o, n in zip(xs, offs, sizes)] + raw, off,
                               SegmentKey(1, 2, 3, 0, 0), out)
        g = (rng.standard_normal(off) * 1e-3).astype(np.float32)
        rs = torch.zeros(off, device=dev)
        comm.reduce_scatter_pieces(torch.from_numpy(g).to(dev),
                                   list(zip(offs, sizes)) + [(o, n, True) for _, o, n, _ in raw], off,
                                   SegmentKey(1, 2, 3, 2, 0), rs)
        o, r = out.cpu().numpy(), rs.cpu().numpy()
        for _, a, n, _ in raw:  # full-precision pieces: copied / averaged over one rank
            assert np.array_equal(o[a:a + n], base[a:a + n].cpu().numpy())
            assert np.array_equal(r[a:a + n], g[a:a + n])
        for x, a, n in zip(xs, offs, sizes):
            c, m, _ = oracle.quantize_segment(x, a, 1024, 8, 0, (1, 2, 3, 0, 0), 8)
            assert np.array_equal(o[a:a + n], oracle.dequantize_segment(c, m, n, 1024, 8, 8).astype(np.float32))
            c, m, _ = oracle.quantize_segment(g[a:a + n], a, 1024, 4, 1, (1, 2, 3, 2, 0), 8)
            exp = (np.zeros(n) + oracle.dequantize_segment(c, m, n, 1024, 4, 8)) / 1
            assert np.array_equal(r[a:a + n], exp.astype(np.float32))
        comm.close()
