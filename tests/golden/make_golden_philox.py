"""Golden vectors for the counter-based noise mode (QSDP_NOISE_PHILOX4x64), from the
LIVE reference quantizer with a numpy Philox generator (dev container only):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_philox.py

Writes tests/golden/golden_philox.npz:

* ph_keys / ph_draws:  raw 64-bit draws of np.random.Philox(SeedSequence(key6))
                       (numpy is the reference's unpinned dependency, pkg/pyproject.toml:9;
                       numpy.__version__ is recorded);
* phq_*:               _segment_blocks(seg, start, S, bits, inner, rng_for_start) with
                       rng_for_start(s) = Generator(Philox(SeedSequence((root, step, layer,
                       phase, worker, s)))) -- the reference's own quantize_bucket
                       (quantize.py:235-286) driven by the Philox generator it accepts
                       (quantize.py:235-241) -- codes (LSB-first packed per bucket,
                       wire.py:82-85), {shift, lo, hi} and dequantize() fp64.

Reuses make_golden.py's input distributions.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import _input  # noqa: E402
from qsdp.quantize import dequantize  # noqa: E402
from qsdp.sharded import _segment_blocks  # noqa: E402
from qsdp.wire import _pack_codes  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_philox.npz")


def philox_rng(key5):
    return lambda s: np.random.Generator(np.random.Philox(np.random.SeedSequence(tuple(key5) + (s,))))


def main():
    rng = np.random.default_rng(2302_02390)
    out = {"numpy_version": np.array(np.__version__)}
    keys, draws = [], []
    for t in range(48):
        k = [int(v) for v in rng.integers(0, 2**32, 6)]
        if t % 4 == 1:
            k[5] = int(rng.integers(2**32, 2**62))  # two-word start
        if t % 4 == 2:
            k[0] = 0
        g = np.random.Philox(np.random.SeedSequence(tuple(k)))
        keys.append(k)
        draws.append([int(v) for v in g.random_raw(9)])
    out["ph_keys"] = np.array(keys, dtype=np.uint64)
    out["ph_draws"] = np.array(draws, dtype=np.uint64)
    cases = []
    for bits, inner in [(8, "shift"), (8, "uniform_stochastic"), (4, "uniform_stochastic"), (6, "shift"),
                        (5, "uniform_stochastic"), (2, "uniform_stochastic")]:
        cases.append((bits, inner, 1024, 3000, 4096, (0, 3, 2, 0 if inner == "shift" else 2, 1), "f32", "normal"))
    for S in (64, 100, 256, 4096):
        cases.append((4, "uniform_stochastic", S, 3 * S + 17, 123457, (7, 1, 4, 2, 3), "f32", "normal"))
        cases.append((8, "shift", S, 2 * S + 5, 999, (7, 1, 4, 1, 0), "f32", "normal"))
    for bits in (1, 3, 8, 12, 16):
        cases.append((bits, "uniform_stochastic", 100, 333, 2**33 + 7, (1, 2, 3, 2, 0), "f64", "normal"))
    cases.append((8, "uniform_stochastic", 1024, 4096, 0, (0, 0, 0, 2, 5), "f32", "constant_mix"))
    cases.append((8, "uniform_stochastic", 1024, 2048, 0, (9, 9, 9, 2, 1), "f32", "student_t"))
    rows = []
    for i, (bits, inner, S, n, start, key, dtype, dist) in enumerate(cases):
        x = _input(n, dtype, dist, rng)
        blocks = _segment_blocks(x, start, S, bits, inner, philox_rng(key))
        packed = np.frombuffer(b"".join(_pack_codes(b.codes, bits) for b in blocks), dtype=np.uint8)
        meta = np.array([[b.shift, b.scale_lo, b.scale_hi] for b in blocks], dtype=np.float32)
        deq = np.concatenate([dequantize(b) for b in blocks])
        out[f"phq_{i}_x"] = x.astype(np.float32) if dtype == "f32" else x
        out[f"phq_{i}_codes"] = packed
        out[f"phq_{i}_meta"] = meta
        out[f"phq_{i}_deq"] = deq
        rows.append((bits, 0 if inner == "shift" else 1, S, n, start) + tuple(key))
    out["phq_cases"] = np.array(rows, dtype=np.int64)
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT}: {len(cases)} quantizer cases, {len(keys)} draw vectors (numpy {np.__version__})")


if __name__ == "__main__":
    main()
