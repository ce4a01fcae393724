"""Golden vectors for the shared-generator bucketing, from the LIVE reference
(dev container only):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_shared.py

Writes tests/golden/golden_shared.npz: for each case the reference's
bucketed_quantize(v, BucketSpec(S), bits, inner, rng=np.random.default_rng(seed))
(quantize.py:289-313) -- one Generator consumed across buckets, no draw for degenerate
buckets -- packed codes (wire.py:82-85), {shift, lo, hi}, dequantize() fp64, and the
generator's next raw output afterwards (where the reference leaves the stream); plus
UniformStochasticGradientQuantizer (optimizer.py:177-191) outputs."""

from __future__ import annotations

import os

import numpy as np
from qsdp.optimizer import UniformStochasticGradientQuantizer
from qsdp.quantize import BucketSpec, LevelTable, bucketed_quantize, dequantize, quantize_with_levels
from qsdp.wire import _pack_codes

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_shared.npz")


def main():
    rng = np.random.default_rng(3_4_2023)
    out = {"numpy_version": np.array(np.__version__)}
    cases = [(8, "uniform_stochastic", 1024, 5000, 1), (8, "shift", 1024, 5000, 2), (4, "uniform_stochastic", 100, 777, 3),
             (3, "shift", 7, 60, 4), (16, "uniform_stochastic", 256, 1000, 5), (8, "uniform_stochastic", 64, 640, 6),
             (8, "shift", 64, 640, 7), (6, "uniform_stochastic", 1024, 4096, 8)]
    rows = []
    for i, (bits, inner, S, n, seed) in enumerate(cases):
        v = rng.standard_normal(n) * 0.02
        if i % 2 == 0:  # degenerate buckets draw nothing: the stream offsets of later buckets move
            v[S:2 * S] = 0.125
            v[n - 3:] = -1.0 if n - 3 >= (n // S) * S else v[n - 3:]
        g = np.random.default_rng(seed)
        blocks = bucketed_quantize(v, BucketSpec(S), bits, inner, rng=g)
        out[f"sh_{i}_x"] = v
        out[f"sh_{i}_codes"] = np.frombuffer(b"".join(_pack_codes(b.codes, bits) for b in blocks), dtype=np.uint8)
        out[f"sh_{i}_meta"] = np.array([[b.shift, b.scale_lo, b.scale_hi] for b in blocks], dtype=np.float32)
        out[f"sh_{i}_deq"] = np.concatenate([dequantize(b) for b in blocks])
        out[f"sh_{i}_next"] = np.array([g.bit_generator.random_raw()], dtype=np.uint64)
        rows.append((bits, 0 if inner == "shift" else 1, S, n, seed))
    out["sh_cases"] = np.array(rows, dtype=np.int64)
    q = UniformStochasticGradientQuantizer(8)
    g = np.random.default_rng(99)
    grad = rng.standard_normal(3000) * 1e-3
    ghat, bits = q(grad, g)
    out.update(usgq_grad=grad, usgq_ghat=ghat, usgq_bits=np.array(bits), usgq_next=np.array([g.bit_generator.random_raw()],
                                                                                             dtype=np.uint64))
    # quantize_with_levels(u, table, stochastic=True, rng) (quantize.py:400-422)
    lv_rows = []
    for k, (nl, n, seed) in enumerate([(16, 5000, 21), (256, 3000, 22), (2, 100, 23), (64, 777, 24)]):
        q = np.sort(rng.uniform(0, 1, nl))
        q[0], q[-1] = 0.0, 1.0
        u = rng.uniform(-0.1, 1.1, n)  # values outside the table's span are clipped
        u[:5] = q[:5] if nl >= 5 else u[:5]  # exactly on levels
        g = np.random.default_rng(seed)
        out[f"lvs_{k}_table"] = q
        out[f"lvs_{k}_u"] = u
        out[f"lvs_{k}_codes"] = quantize_with_levels(u, LevelTable(q), stochastic=True, rng=g)
        out[f"lvs_{k}_next"] = np.array([g.bit_generator.random_raw()], dtype=np.uint64)
        lv_rows.append(seed)
    out["lvs_seeds"] = np.array(lv_rows, dtype=np.int64)
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT}: {len(cases)} cases")


if __name__ == "__main__":
    main()
