"""GPU parity: K1/K2/K3/K4 through the C ABI vs the reference's golden vectors
and the oracle.  Bar: codes and scales bit-exact; fp64 dequant bit-exact;
fp32 dequant == float32(reference fp64) bit-exact; bf16 == bf16(fp32 output)."""

import numpy as np
import pytest
import torch

from conftest import golden_cases
from paper_2302_02390_b200.quantize import (QuantSpec, SegmentKey, codes_bytes, dequant_accumulate,
                                            dequantize_segment, quantize_segment, quantize_segments)

pytestmark = pytest.mark.gpu
INNER = {0: "shift", 1: "uniform_stochastic"}


def _dev():
    return torch.device("cuda", 0)


def _q(x_np, start, spec, key, dtype=None):
    x = torch.from_numpy(np.ascontiguousarray(x_np if dtype is None else x_np.astype(dtype))).to(_dev())
    codes, meta = quantize_segment(x, start, spec, SegmentKey(*key))
    return codes.cpu().numpy(), meta.cpu().numpy()


def test_golden_codes_scales_dequant(golden):
    for c in golden_cases(golden):
        spec = QuantSpec(c["bits"], c["bucket"], INNER[c["inner"]])
        codes, meta = _q(c["x"], c["start"], spec, c["key"])
        assert np.array_equal(codes, c["codes"]), c["i"]
        assert np.array_equal(meta, c["meta"]), c["i"]
        # also bit-identical meta words (sign of zero included)
        assert np.array_equal(meta.view(np.uint32), c["meta"].view(np.uint32)), c["i"]
        dc = torch.from_numpy(codes).to(_dev())
        dm = torch.from_numpy(meta).to(_dev())
        d64 = dequantize_segment(dc, dm, c["n"], spec, dtype=torch.float64).cpu().numpy()
        assert np.array_equal(d64, c["deq"]), c["i"]
        d32 = dequantize_segment(dc, dm, c["n"], spec, dtype=torch.float32).cpu().numpy()
        assert np.array_equal(d32.view(np.uint32), c["deq"].astype(np.float32).view(np.uint32)), c["i"]
        db = dequantize_segment(dc, dm, c["n"], spec, dtype=torch.bfloat16)
        assert torch.equal(db.cpu(), torch.from_numpy(d32).to(torch.bfloat16)), c["i"]


@pytest.mark.parametrize("bits,inner", [(8, 0), (8, 1), (4, 1), (4, 0), (6, 0), (5, 1), (2, 1), (16, 0),
                                        (1, 0), (3, 1)])
@pytest.mark.parametrize("bucket", [64, 1024, 4096])
def test_random_vs_oracle(oracle, bits, inner, bucket):
    rng = np.random.default_rng(bits * 100 + inner * 7 + bucket)
    n = 3 * bucket * 7 + 5
    x = (rng.standard_normal(n) * 0.02).astype(np.float32)
    key = (11, 5, 3, 2 if inner else 1, 6)
    start = int(rng.integers(0, 2**40))
    spec = QuantSpec(bits, bucket, INNER[inner])
    codes, meta = _q(x, start, spec, key)
    oc, om, _ = oracle.quantize_segment(x, start, bucket, bits, inner, key, 8)
    assert np.array_equal(codes, oc)
    assert np.array_equal(meta.view(np.uint32), om.view(np.uint32))


@pytest.mark.parametrize("inner,bits", [(0, 8), (1, 8), (1, 4)])
def test_large_segment_vs_oracle(oracle, inner, bits):
    """2^23 GPT-like weights (and heavy-tailed gradients): codes bit-exact."""
    rng = np.random.default_rng(inner * 10 + bits)
    n = 1 << 23
    x = (rng.standard_t(3, n) * (0.02 if inner == 0 else 1e-3)).astype(np.float32)
    key = (0, 17, 9, 2 if inner else 0, 3)
    spec = QuantSpec(bits, 1024, INNER[inner])
    codes, meta = _q(x, 1 << 20, spec, key)
    oc, om, _ = oracle.quantize_segment(x, 1 << 20, 1024, bits, inner, key, 8)
    assert np.array_equal(meta.view(np.uint32), om.view(np.uint32))
    mism = np.flatnonzero(codes != oc)
    assert mism.size == 0, f"{mism.size} code bytes differ, first at {mism[:5]}"


@pytest.mark.parametrize("bits", [8, 4, 2, 1])
def test_shift_fp32_certificate_stress(oracle, bits):
    """K1's fp32-certified fast path against the oracle on 2^21 elements per
    distribution: grid-valued data (many exact ties), tiny and huge spans on both sides of the
    fp32 guard, zero extrema of either sign, subnormals."""
    rng = np.random.default_rng(bits)
    n = 1 << 21
    dists = {
        "grid": np.floor(rng.uniform(0, 256, n)) / 255.0,
        "uniform": rng.uniform(-1, 1, n),
        "tiny_span": 1.0 + rng.uniform(0, 1, n) * 2.0 ** -20,
        "subnormal": rng.uniform(0, 1, n) * 1e-40,
        "span_near_guard": rng.uniform(-1, 1, n) * 2.0 ** 99,
        "span_beyond_guard": rng.uniform(-1, 1, n) * 2.0 ** 120,
        "small_beyond_guard": rng.uniform(0, 1, n) * 2.0 ** -110,
        "zero_extrema": np.where(rng.uniform(size=n) < 0.5, rng.uniform(0, 1, n), 0.0) *
                        np.where(np.arange(n) % 2048 < 1024, 1.0, -1.0),
    }
    dists["zero_extrema"][::7] = -0.0
    for name, x in dists.items():
        x = x.astype(np.float32)
        key = (3, 1, 4, 1, 5)
        spec = QuantSpec(bits, 1024, "shift")
        codes, meta = _q(x, 12345, spec, key)
        oc, om, _ = oracle.quantize_segment(x, 12345, 1024, bits, 0, key, 8)
        mism = np.flatnonzero(codes != oc)
        assert mism.size == 0, (name, mism.size, mism[:5])
        assert np.array_equal(meta, om), name


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_edge_lengths_and_alignment(oracle, dtype):
    """Short / empty-ish segments, misaligned starts (scalar path), odd buckets (generic path)."""
    rng = np.random.default_rng(5)
    base = rng.standard_normal(5000).astype(dtype)
    for bucket in (8, 64, 100, 7, 1024):
        for n in (1, 3, 7, 8, 9, 63, 1025, 2049):
            for off in (0, 1, 3):
                x_full = torch.from_numpy(base).to(_dev())
                x = x_full[off:off + n]  # possibly not 16B aligned
                for inner in (0, 1):
                    spec = QuantSpec(8 if inner == 0 else 4, bucket, INNER[inner])
                    key = SegmentKey(1, 2, 3, 2 if inner else 0, 1)
                    codes, meta = quantize_segment(x, 77 + off, spec, key)
                    oc, om, _ = oracle.quantize_segment(base[off:off + n].astype(np.float64), 77 + off,
                                                        bucket, spec.bits, inner, (1, 2, 3, 2 if inner else 0, 1))
                    assert np.array_equal(codes.cpu().numpy(), oc), (bucket, n, off, inner)
                    assert np.array_equal(meta.cpu().numpy(), om), (bucket, n, off, inner)
                    out = torch.empty(n + 1, dtype=torch.float64, device=_dev())[1:]  # misaligned output
                    dequantize_segment(codes, meta, n, spec, dtype=torch.float64, out=out)
                    assert np.array_equal(out.cpu().numpy(),
                                          oracle.dequantize_segment(oc, om, n, bucket, spec.bits))


def test_degenerate_and_special_values(oracle):
    x = np.zeros(4096, dtype=np.float32)
    x[1024:2048] = 0.25
    x[2048:3072] = -0.0
    x[3072:] = np.float32(3.4e38) * np.where(np.arange(1024) % 2, 1, -1)  # huge range
    x[5] = 1e-45  # denormal
    for inner in (0, 1):
        spec = QuantSpec(8, 1024, INNER[inner])
        codes, meta = _q(x, 0, spec, (0, 0, 0, 0, 0))
        oc, om, _ = oracle.quantize_segment(x, 0, 1024, 8, inner, (0, 0, 0, 0, 0))
        assert np.array_equal(codes, oc)
        assert np.array_equal(meta.view(np.uint32), om.view(np.uint32))


def test_nonfinite_raises_with_index():
    x = torch.zeros(5000, device=_dev())
    x[3001] = float("inf")
    x[4000] = float("nan")
    with pytest.raises(ValueError, match="index 3001"):
        quantize_segment(x, 0, QuantSpec(8, 1024, "shift"), SegmentKey(), check_finite=True)


def test_batched_segments_equal_individual(oracle):
    rng = np.random.default_rng(9)
    xs = [torch.from_numpy(rng.standard_normal(n).astype(np.float32)).to(_dev()) for n in (5000, 1024, 17, 70000)]
    spec = QuantSpec(8, 1024, "uniform_stochastic")
    items = [(x, 1000 * i, SegmentKey(3, 1, i, 2, i)) for i, x in enumerate(xs)]
    batched = quantize_segments(items, spec)
    for it, (c, m) in zip(items, batched):
        c1, m1 = quantize_segment(*it[:2], spec, it[2])
        assert torch.equal(c, c1) and torch.equal(m, m1)


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("bits", [8, 4])
def test_dequant_accumulate_vs_oracle(oracle, P, bits):
    rng = np.random.default_rng(P * 31 + bits)
    n = 10 * 1024 + 300
    grads = [(rng.standard_normal(n) * 1e-3) for _ in range(P)]
    spec = QuantSpec(bits, 1024, "uniform_stochastic")
    srcs = []
    for p in range(P):
        x = torch.from_numpy(grads[p]).to(_dev())
        srcs.append(quantize_segment(x, 4096, spec, SegmentKey(0, 3, 7, 2, p)))
    out64 = dequant_accumulate(srcs, n, spec, P, dtype=torch.float64).cpu().numpy()
    out32 = dequant_accumulate(srcs, n, spec, P, dtype=torch.float32).cpu().numpy()
    acc = np.zeros(n)
    for p in range(P):
        c, m, _ = oracle.quantize_segment(grads[p], 4096, 1024, bits, 1, (0, 3, 7, 2, p))
        acc = acc + oracle.dequantize_segment(c, m, n, 1024, bits)
    ref = acc / P
    assert np.array_equal(out64, ref)
    assert np.array_equal(out32.view(np.uint32), ref.astype(np.float32).view(np.uint32))


def test_deterministic_across_runs():
    x = torch.randn(1 << 20, device=_dev())
    spec = QuantSpec(8, 1024, "uniform_stochastic")
    a = quantize_segment(x, 0, spec, SegmentKey(1, 2, 3, 2, 0))
    b = quantize_segment(x, 0, spec, SegmentKey(1, 2, 3, 2, 0))
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
    c = quantize_segment(x, 0, spec, SegmentKey(1, 2, 3, 2, 1))  # other worker -> other noise
    assert not torch.equal(a[0], c[0])


def test_codes_buffer_size():
    spec = QuantSpec(5, 64, "shift")
    x = torch.randn(1000, device=_dev())
    c, m = quantize_segment(x, 0, spec, SegmentKey())
    assert c.numel() == codes_bytes(1000, spec) == 15 * 40 + 25
    assert m.shape == (16, 3)


def test_reference_api_mirror(golden):
    """quantize_bucket / bucketed_quantize / dequantize with bucket_rng keys."""
    from paper_2302_02390_b200.quantize import BucketSpec, bucket_rng, bucketed_quantize, dequantize, \
        quantize_bucket
    c = next(cc for cc in golden_cases(golden) if cc["bucket"] == 1024 and cc["n"] == 3000)
    mode = INNER[c["inner"]]
    blocks = bucketed_quantize(c["x"].astype(np.float64), BucketSpec(1024), c["bits"], mode,
                               bucket_rng(*c["key"], c["start"]))
    deq = np.concatenate([dequantize(b, mode) for b in blocks])
    assert np.array_equal(deq, c["deq"])
    b0 = quantize_bucket(c["x"][:1024].astype(np.float64), c["bits"], mode, bucket_rng(*c["key"], c["start"]))
    assert b0 == blocks[0]
    # KATs: test_quantize.py:229-234 (constant bucket) and :291-295 (on-level stochastic codes)
    blk = quantize_bucket(np.full(10, 0.3), 8, "shift", bucket_rng(0, 0, 0, 0, 0, 0))
    assert blk.scale_lo == blk.scale_hi and np.all(dequantize(blk) == np.float32(0.3))
    blk = quantize_bucket(np.array([0.0, 1 / 15, 1.0]), 4, "uniform_stochastic", bucket_rng(0, 0, 0, 2, 0, 0))
    assert list(blk.codes) == [0, 1, 15]
    with pytest.raises(ValueError, match="non-finite"):
        quantize_bucket(np.array([1.0, np.nan]), 8, "shift", bucket_rng(0, 0, 0, 0, 0, 0))
    with pytest.raises(ValueError, match="corrupted"):
        from paper_2302_02390_b200.quantize import QuantizedBlock
        bad = QuantizedBlock(np.array([3]), 0.0, 0.0, 1.0, 2, 1)
        bad.codes = np.array([7], dtype=np.uint32)
        dequantize(bad)
