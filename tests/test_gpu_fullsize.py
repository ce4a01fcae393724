"""GPU: the bench's full GPT-2 125M step (BASELINE.json configs[1]: 13 FSDP groups, 124.3 M
dense parameters, w8/g8, bucket 1024) through the communicator at world 1, checked with
size-independent properties on every element plus bit-exact oracle checks on sampled buckets:

* all-gather (random shift, quantize.py:265-271): |x_hat - x| <= pitch / 2 per bucket, pitch =
  (hi - lo) / top (plus the fp32 output rounding);
* reduce-scatter (stochastic, quantize.py:316-321): |x_hat - x| < pitch, and the rounding is
  unbiased over the tensor (mean error within 6 standard errors of 0);
* the scales: lo / hi are the fp32 bucket min / max, so every x lies in [lo, hi];
* 32 random buckets per group and kind, and every group's partial last bucket, equal the
  oracle's dequantized values bit for bit."""

import numpy as np
import pytest
import torch

from paper_2302_02390_b200.comm import QSDPComm
from paper_2302_02390_b200.gpt import dense_groups
from paper_2302_02390_b200.quantize import QuantSpec, SegmentKey

pytestmark = pytest.mark.gpu

S, BITS = 1024, 8
TOP = (1 << BITS) - 1


def _bucket_bounds(x: torch.Tensor):
    nf = x.numel() // S
    xb = x[:nf * S].view(nf, S).double()
    lo = xb.min(dim=1).values.float().double()  # _f32(min), _f32(max)
    hi = xb.max(dim=1).values.float().double()
    return xb, lo, hi, (hi - lo) / TOP


def test_gpt2_small_step_properties_and_sampled_parity(oracle):
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev).manual_seed(2024)
    rng = np.random.default_rng(5)
    groups = dense_groups("gpt2-125m")
    assert sum(g.numel for g in groups) == 124318464
    comm = QSDPComm(max(g.numel for g in groups), QuantSpec(BITS, S, "shift"),
                    QuantSpec(BITS, S, "uniform_stochastic"), device=dev)
    for gi, g in enumerate(groups):
        n = g.numel
        x = torch.randn(n, generator=gen, device=dev) * 0.02
        gr = torch.randn(n, generator=gen, device=dev) * 1e-3
        full = torch.empty(n, device=dev)
        shard = torch.empty(n, device=dev)
        comm.all_gather(x, [(0, n)], SegmentKey(0, 3, gi, 0, 0), full)
        comm.reduce_scatter(gr, [(0, n)], SegmentKey(0, 3, gi, 2, 0), shard)
        torch.cuda.synchronize()
        nf = n // S
        for kind, src, out in (("ag", x, full), ("rs", gr, shard)):
            xb, lo, hi, pitch = _bucket_bounds(src)
            yb = out[:nf * S].view(nf, S).double()
            err = (yb - xb).abs()
            slack = 1e-6 * pitch[:, None] + 2.0 ** -23 * yb.abs()  # fp32 output rounding
            bound = pitch[:, None] * (0.5 if kind == "ag" else 1.0)
            assert bool((err <= bound + slack).all()), (gi, kind, float((err - bound).max()))
            assert bool(((xb >= lo[:, None]) & (xb <= hi[:, None])).all())
            if kind == "rs":  # unbiased stochastic rounding: E[x_hat - x] = 0
                d = (yb - xb).flatten()
                se = float(pitch.mean()) / np.sqrt(d.numel())
                assert abs(float(d.mean())) < 6 * se, (gi, float(d.mean()), se)
            # sampled buckets (and the partial last one) bit-exact against the oracle
            xs, ys = src.cpu().numpy(), out.cpu().numpy()
            nb = (n + S - 1) // S
            picks = sorted(set(rng.choice(nb, size=min(32, nb), replace=False).tolist()) | {nb - 1})
            inner, phase = (0, 0) if kind == "ag" else (1, 2)
            for b in picks:
                a, e = b * S, min(n, (b + 1) * S)
                c, m, _ = oracle.quantize_segment(xs[a:e], a, S, BITS, inner, (0, 3, gi, phase, 0), 1)
                exp = oracle.dequantize_segment(c, m, e - a, S, BITS, 1).astype(np.float32)
                assert np.array_equal(ys[a:e], exp), (gi, kind, b)
    comm.close()


def test_two_gigabyte_tensor_sampled_parity(oracle):
    """A 2^29 + 1000-element (2 GB fp32) tensor -- past the top of the SURVEY §8(d) sweep --
    through one all-gather / reduce-scatter: input byte offsets past 2^31 (64-bit indexing
    everywhere), checked on sampled buckets across the whole range, the last ones included."""
    dev = torch.device("cuda", 0)
    n = (1 << 29) + 1000
    gen = torch.Generator(device=dev).manual_seed(7)
    comm = QSDPComm(n, QuantSpec(BITS, S, "shift"), QuantSpec(4, S, "uniform_stochastic"), device=dev)
    x = torch.randn(n, generator=gen, device=dev) * 0.02
    out = torch.empty(n, device=dev)
    comm.all_gather(x, [(0, n)], SegmentKey(1, 9, 2, 1, 0), out)
    sh = torch.empty(n, device=dev)
    comm.reduce_scatter(x, [(0, n)], SegmentKey(1, 9, 2, 2, 0), sh)
    torch.cuda.synchronize()
    nb = (n + S - 1) // S
    rng = np.random.default_rng(3)
    picks = sorted(set(rng.choice(nb, size=48, replace=False).tolist()) | {0, nb // 2, nb - 2, nb - 1})
    for b in picks:
        a, e = b * S, min(n, (b + 1) * S)
        xs = x[a:e].cpu().numpy()
        for inner, bits, phase, y in ((0, BITS, 1, out), (1, 4, 2, sh)):
            c, m, _ = oracle.quantize_segment(xs, a, S, bits, inner, (1, 9, 2, phase, 0), 1)
            exp = oracle.dequantize_segment(c, m, e - a, S, bits, 1).astype(np.float32)
            assert np.array_equal(y[a:e].cpu().numpy(), exp), (b, inner)
    comm.close()
