"""GPU: bucketed quantization with ONE numpy Generator shared by the buckets (the reference's
bucketed_quantize with an rng, quantize.py:289-313, and the theory side's
UniformStochasticGradientQuantizer, optimizer.py:177-191): codes, scales and the
generator's final state bit-exact vs the reference goldens; degenerate buckets draw nothing."""

import os

import numpy as np
import pytest

from paper_2302_02390_b200.quantize import BucketSpec, bucketed_quantize, dequantize, quantize_bucket

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(__file__), "golden", "golden_shared.npz")


def _pack(blocks, bits):
    from paper_2302_02390_b200.quantize import _pack
    return np.concatenate([_pack(b.codes, bits) for b in blocks])


def test_shared_generator_golden():
    g = np.load(G)
    for i, (bits, inner, S, n, seed) in enumerate(g["sh_cases"]):
        rng = np.random.default_rng(int(seed))
        blocks = bucketed_quantize(g[f"sh_{i}_x"], BucketSpec(int(S)), int(bits),
                                   "shift" if inner == 0 else "uniform_stochastic", rng=rng)
        assert np.array_equal(_pack(blocks, int(bits)), g[f"sh_{i}_codes"]), i
        meta = np.array([[b.shift, b.scale_lo, b.scale_hi] for b in blocks], dtype=np.float32)
        assert np.array_equal(meta, g[f"sh_{i}_meta"]), i
        assert np.array_equal(np.concatenate([dequantize(b) for b in blocks]), g[f"sh_{i}_deq"]), i
        assert int(rng.bit_generator.random_raw()) == int(g[f"sh_{i}_next"][0]), i  # the stream left where numpy leaves it


def test_uniform_stochastic_gradient_quantizer_dropin():
    """optimizer.py:184-191's body with the product's bucketed_quantize / dequantize."""
    g = np.load(G)
    rng = np.random.default_rng(99)
    blocks = bucketed_quantize(g["usgq_grad"], BucketSpec(), 8, inner="uniform_stochastic", rng=rng)
    ghat = np.concatenate([dequantize(b, "uniform_stochastic") for b in blocks])
    assert np.array_equal(ghat, g["usgq_ghat"])
    assert int(rng.bit_generator.random_raw()) == int(g["usgq_next"][0])


def test_shared_generator_vs_oracle_and_errors(oracle):
    rng0 = np.random.default_rng(5)
    v = rng0.standard_normal(10_000) * 0.02
    v[3000:4000] = 0.5
    for bits, inner, S in ((8, "uniform_stochastic", 1000), (5, "shift", 333), (2, "uniform_stochastic", 64)):
        rng = np.random.default_rng(17)
        st = rng.bit_generator.state["state"]
        blocks = bucketed_quantize(v, BucketSpec(S), bits, inner, rng=rng)
        oc, om, bad, (s2, _) = oracle.quantize_shared(v, S, bits, 0 if inner == "shift" else 1, int(st["state"]),
                                                      int(st["inc"]))
        assert bad == -1 and np.array_equal(_pack(blocks, bits), oc)
        assert int(rng.bit_generator.state["state"]["state"]) == s2
    # one bucket through quantize_bucket continues the stream too
    rng = np.random.default_rng(3)
    b1 = quantize_bucket(v[:1024], 8, "uniform_stochastic", rng)
    b2 = quantize_bucket(v[1024:2048], 8, "uniform_stochastic", rng)
    both = bucketed_quantize(v[:2048], BucketSpec(1024), 8, "uniform_stochastic", rng=np.random.default_rng(3))
    assert np.array_equal(b1.codes, both[0].codes) and np.array_equal(b2.codes, both[1].codes)
    # a non-finite value raises like _check_finite after the earlier buckets consumed their draws
    w = v.copy()
    w[2500] = np.nan
    rng = np.random.default_rng(8)
    with pytest.raises(ValueError, match="non-finite bucket value at index 500"):
        bucketed_quantize(w, BucketSpec(1000), 8, "uniform_stochastic", rng=rng)
    ref = np.random.default_rng(8)
    ref.bit_generator.advance(2000)
    assert int(rng.bit_generator.random_raw()) == int(ref.bit_generator.random_raw())


def test_stochastic_levels_golden():
    """quantize_with_levels(u, table, stochastic=True, rng) (quantize.py:400-422) on the device:
    codes and the generator's final state equal the reference's."""
    from paper_2302_02390_b200.levels import LevelTable, quantize_with_levels
    g = np.load(G)
    for k, seed in enumerate(g["lvs_seeds"]):
        rng = np.random.default_rng(int(seed))
        codes = quantize_with_levels(g[f"lvs_{k}_u"], LevelTable(g[f"lvs_{k}_table"]), stochastic=True, rng=rng)
        assert np.array_equal(codes, g[f"lvs_{k}_codes"]), k
        assert int(rng.bit_generator.random_raw()) == int(g[f"lvs_{k}_next"][0]), k
