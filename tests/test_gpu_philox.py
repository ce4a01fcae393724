"""GPU parity of the counter-based noise mode (QSDP_NOISE_PHILOX4x64): the quantizers
driven by numpy's Philox4x64-10 keyed like bucket_rng, i.e. the reference's
quantize_bucket with Generator(Philox(SeedSequence(key))) (quantize.py:235-241).
Bar: codes and scales bit-exact vs the reference goldens and the oracle."""

import numpy as np
import pytest
import torch

from conftest import golden_philox_cases
from paper_2302_02390_b200.quantize import (QuantSpec, SegmentKey, bucketed_quantize, BucketSpec, dequantize_segment,
                                            philox_rng, quantize_bucket, quantize_segment)

pytestmark = pytest.mark.gpu
INNER = {0: "shift", 1: "uniform_stochastic"}


def _dev():
    return torch.device("cuda", 0)


def test_philox_golden(golden_philox):
    for c in golden_philox_cases(golden_philox):
        spec = QuantSpec(c["bits"], c["bucket"], INNER[c["inner"]], "philox")
        x = torch.from_numpy(np.ascontiguousarray(c["x"])).to(_dev())
        codes, meta = quantize_segment(x, c["start"], spec, SegmentKey(*c["key"]))
        assert np.array_equal(codes.cpu().numpy(), c["codes"]), c["i"]
        assert np.array_equal(meta.cpu().numpy().view(np.uint32), c["meta"].view(np.uint32)), c["i"]
        d64 = dequantize_segment(codes, meta, c["n"], spec, dtype=torch.float64).cpu().numpy()
        assert np.array_equal(d64, c["deq"]), c["i"]


@pytest.mark.parametrize("bits,inner", [(8, 1), (4, 1), (8, 0), (16, 1), (3, 1), (1, 0)])
@pytest.mark.parametrize("bucket", [24, 100, 1024, 4096])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_philox_random_vs_oracle(oracle, bits, inner, bucket, dtype):
    rng = np.random.default_rng(bits * 31 + inner * 7 + bucket)
    n = 5 * bucket + 13
    x = (rng.standard_normal(n) * 0.02).astype(dtype)
    key = (3, 8, 1, 2 if inner else 0, 5)
    start = int(rng.integers(0, 2**40))
    spec = QuantSpec(bits, bucket, INNER[inner], "philox")
    codes, meta = quantize_segment(torch.from_numpy(x).to(_dev()), start, spec, SegmentKey(*key))
    oc, om, _ = oracle.quantize_segment(x, start, bucket, bits, inner, key, 8, noise=1)
    assert np.array_equal(codes.cpu().numpy(), oc)
    assert np.array_equal(meta.cpu().numpy().view(np.uint32), om.view(np.uint32))


def test_philox_differs_from_pcg64_and_mirror_api(oracle):
    """philox_rng(...) drives the mirrored quantize_bucket / bucketed_quantize; the draws
    are not bucket_rng's (a different stream of the same key)."""
    rng = np.random.default_rng(4)
    v = rng.standard_normal(3000) * 0.02
    blk = quantize_bucket(v[:1024], 8, "uniform_stochastic", philox_rng(1, 2, 3, 2, 0, 77))
    oc, om, _ = oracle.quantize_segment(v[:1024], 77, 1024, 8, 1, (1, 2, 3, 2, 0), 1, noise=1)
    assert np.array_equal(blk.codes, oracle.unpack(oc, 1024, 8))
    pc, _, _ = oracle.quantize_segment(v[:1024], 77, 1024, 8, 1, (1, 2, 3, 2, 0), 1, noise=0)
    assert not np.array_equal(oc, pc)
    blocks = bucketed_quantize(v, BucketSpec(1024), 4, "uniform_stochastic", philox_rng(1, 2, 3, 2, 0, 5))
    oc, om, _ = oracle.quantize_segment(v, 5, 1024, 4, 1, (1, 2, 3, 2, 0), 1, noise=1)
    got = np.concatenate([b.codes for b in blocks])
    assert np.array_equal(got, oracle.unpack(oc, 3000, 4))


def test_philox_collectives_world1(oracle):
    """C1/C2 through the communicator with Philox specs (the TMA fast paths are PCG64-only:
    the collectives take the team kernels plus a separate K3/K4)."""
    from paper_2302_02390_b200.comm import QSDPComm
    dev = _dev()
    size = 1024 * 50 + 7
    ws, gs = QuantSpec(8, 1024, "shift", "philox"), QuantSpec(4, 1024, "uniform_stochastic", "philox")
    comm = QSDPComm(size, ws, gs, device=dev)
    x = (np.random.default_rng(9).standard_normal(size) * 0.02).astype(np.float32)
    xt = torch.from_numpy(x).to(dev)
    out = torch.empty(size, device=dev)
    comm.all_gather(xt, [(0, size)], SegmentKey(0, 4, 1, 0, 0), out)
    c, m, _ = oracle.quantize_segment(x, 0, 1024, 8, 0, (0, 4, 1, 0, 0), 8, noise=1)
    assert np.array_equal(out.cpu().numpy(), oracle.dequantize_segment(c, m, size, 1024, 8, 8).astype(np.float32))
    sh = torch.empty(size, device=dev)
    comm.reduce_scatter(xt, [(0, size)], SegmentKey(0, 4, 1, 2, 0), sh)
    c, m, _ = oracle.quantize_segment(x, 0, 1024, 4, 1, (0, 4, 1, 2, 0), 8, noise=1)
    exp = (np.zeros(size) + oracle.dequantize_segment(c, m, size, 1024, 4, 8)) / 1
    assert np.array_equal(sh.cpu().numpy(), exp.astype(np.float32))
    comm.close()
