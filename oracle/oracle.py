"""TEST INFRASTRUCTURE ONLY -- ctypes front end of the C oracle (qsdp_oracle.c).

The oracle is the CPU restatement of the reference QSDP hot path used to check
the CUDA path.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` leg of ``bench.py`` may import this
module; the product package never does.

Protocol-level helpers restate the reference's simulated collectives:

* :func:`gather` -- ``ShardedMLP._gather`` (pkg/src/qsdp/sharded.py:323-373) /
  ``ReferenceMLP._quantized_view`` (sharded.py:530-550);
* :func:`reduce_scatter` -- ``ShardedMLP._reduce_scatter`` (sharded.py:375-433) /
  ``ReferenceMLP._averaged_gradient`` (sharded.py:552-582).

Parity is pinned by ``tests/golden`` (vectors from the live reference) and, when
``/root/reference`` is mounted, by the live reference itself.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libqsdp_oracle.so")

SHIFT = 0
STOCHASTIC = 1
PHASE_W_FWD = 0
PHASE_W_BWD = 1
PHASE_GRAD = 2

_lib = None


def build() -> str:
    """Compile the oracle with its Makefile (gcc only)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        i64, u64, i32 = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int
        vp = ctypes.c_void_p
        L.qo_seedseq_state.argtypes = [vp, i32, vp]
        L.qo_pcg64_seed.argtypes = [vp, vp]
        L.qo_pcg64_next.argtypes = [vp]
        L.qo_pcg64_next.restype = u64
        L.qo_next_double.argtypes = [vp]
        L.qo_next_double.restype = ctypes.c_double
        L.qo_bucket_rng.argtypes = [vp, u64, u64, u64, u64, u64, u64]
        L.qo_quantize_bucket.argtypes = [vp, i64, i32, i32, vp, vp, vp]
        L.qo_quantize_bucket.restype = i64
        L.qo_dequantize.argtypes = [vp, i64, i32, vp, vp]
        L.qo_pack.argtypes = [vp, i64, i32, vp]
        L.qo_unpack.argtypes = [vp, i64, i32, vp]
        L.qo_unpack.restype = i32
        L.qo_num_buckets.argtypes = [i64, i64]
        L.qo_num_buckets.restype = i64
        L.qo_codes_bytes.argtypes = [i64, i64, i32]
        L.qo_codes_bytes.restype = i64
        qargs = [vp, i64, i64, i64, i32, i32, u64, u64, u64, u64, u64, vp, vp, i32]
        L.qo_quantize_segment.argtypes = qargs
        L.qo_quantize_segment.restype = i64
        L.qo_quantize_segment_f32.argtypes = qargs
        L.qo_quantize_segment_nz.argtypes = qargs + [i32]
        L.qo_quantize_segment_nz.restype = i64
        L.qo_quantize_segment_f32_nz.argtypes = qargs + [i32]
        L.qo_quantize_segment_f32_nz.restype = i64
        L.qo_philox_rng.argtypes = [vp, u64, u64, u64, u64, u64, u64]
        L.qo_quantize_shared.argtypes = [vp, i64, i64, i32, i32, vp, vp, vp]
        L.qo_quantize_shared.restype = i64
        L.qo_philox_next.argtypes = [vp]
        L.qo_philox_next.restype = u64
        L.qo_quantize_segment_f32.restype = i64
        L.qo_dequantize_segment.argtypes = [vp, vp, i64, i64, i32, vp, i32]
        L.qo_dequantize_segment.restype = i32
        L.qo_message_size_bits.argtypes = [i64, i64, i32]
        L.qo_message_size_bits.restype = i64
        L.qo_encode_segment.argtypes = [vp, vp, i64, i64, i32, vp]
        L.qo_encode_segment.restype = i64
        dbl = ctypes.c_double
        L.qo_level_code.argtypes = [dbl, vp, i64]
        L.qo_level_code.restype = ctypes.c_uint32
        L.qo_quantize_levels_segment.argtypes = [vp, i64, i64, i32, vp, vp, vp]
        L.qo_quantize_levels_segment.restype = i64
        L.qo_dequantize_levels_segment.argtypes = [vp, vp, i64, i64, i32, vp, vp]
        L.qo_dequantize_levels_segment.restype = i32
        L.qo_learn_levels.argtypes = [vp, i64, vp, i64, dbl]
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


# -- noise ---------------------------------------------------------------------


def seedseq_state(fields) -> np.ndarray:
    f = np.ascontiguousarray(fields, dtype=np.uint64)
    out = np.zeros(4, dtype=np.uint64)
    lib().qo_seedseq_state(_ptr(f), f.size, _ptr(out))
    return out


class PCG64:
    """Restated numpy PCG64 stream keyed like ``bucket_rng`` (sharded.py:235-240)."""

    def __init__(self, root, step, layer, phase, worker, start):
        self._st = np.zeros(4, dtype=np.uint64)
        lib().qo_bucket_rng(_ptr(self._st), root, step, layer, phase, worker, start)

    def next_raw(self) -> int:
        return int(lib().qo_pcg64_next(_ptr(self._st)))

    def random(self) -> float:
        return float(lib().qo_next_double(_ptr(self._st)))


class Philox:
    """Restated numpy Philox4x64-10 stream: Generator(Philox(SeedSequence(key6)))."""

    def __init__(self, root, step, layer, phase, worker, start):
        self._st = np.zeros(16, dtype=np.uint64)  # qo_philox: ctr[4], key[2], buf[4], pos
        lib().qo_philox_rng(_ptr(self._st), root, step, layer, phase, worker, start)

    def next_raw(self) -> int:
        return int(lib().qo_philox_next(_ptr(self._st)))

    def random(self) -> float:
        return (self.next_raw() >> 11) * 2.0 ** -53


NOISE = {"pcg64": 0, "philox": 1}


def quantize_shared(v, bucket, bits, inner, state: int, inc: int):
    """bucketed_quantize with one shared numpy PCG64 stream (quantize.py:289-313) from
    (state, inc); returns (packed codes, meta, bad index, final (state, inc))."""
    v = np.ascontiguousarray(v, dtype=np.float64)
    n = v.size
    g = np.array([state >> 64, state & (2**64 - 1), inc >> 64, inc & (2**64 - 1)], dtype=np.uint64)
    codes = np.zeros(max(codes_bytes(n, bucket, bits), 1), dtype=np.uint8)
    meta = np.zeros((max(num_buckets(n, bucket), 1), 3), dtype=np.float32)
    bad = lib().qo_quantize_shared(_ptr(v), n, bucket, bits, inner, _ptr(g), _ptr(codes), _ptr(meta))
    return (codes[: codes_bytes(n, bucket, bits)], meta[: num_buckets(n, bucket)], int(bad),
            ((int(g[0]) << 64) | int(g[1]), (int(g[2]) << 64) | int(g[3])))


# -- per-bucket / per-segment quantizer -------------------------------------------


def num_buckets(length: int, bucket: int) -> int:
    return int(lib().qo_num_buckets(length, bucket))


def codes_bytes(length: int, bucket: int, bits: int) -> int:
    return int(lib().qo_codes_bytes(length, bucket, bits))


def message_size_bits(length: int, bucket: int, bits: int) -> int:
    return int(lib().qo_message_size_bits(length, bucket, bits))


def quantize_segment(x, global_start, bucket, bits, inner, key, nthreads=1, noise=0):
    """Returns (packed codes uint8, meta float32[nb,3] = shift, lo, hi, bad_index).

    ``key`` = (root_seed, step, layer, phase, worker); bucket j is keyed with
    start = global_start + j*bucket (sharded.py:243-248).  ``noise`` 0: PCG64
    (bucket_rng), 1: Philox4x64-10 with the same SeedSequence key.
    """
    x = np.ascontiguousarray(x)
    n = x.size
    codes = np.zeros(max(codes_bytes(n, bucket, bits), 1), dtype=np.uint8)
    meta = np.zeros((max(num_buckets(n, bucket), 1), 3), dtype=np.float32)
    fn = lib().qo_quantize_segment_f32_nz if x.dtype == np.float32 else lib().qo_quantize_segment_nz
    if x.dtype != np.float32:
        x = np.ascontiguousarray(x, dtype=np.float64)
    root, step, layer, phase, worker = key
    bad = fn(_ptr(x), n, global_start, bucket, bits, inner, root, step, layer, phase, worker,
             _ptr(codes), _ptr(meta), nthreads, int(noise))
    return codes[: codes_bytes(n, bucket, bits)], meta[: num_buckets(n, bucket)], int(bad)


def dequantize_segment(codes, meta, length, bucket, bits, nthreads=1) -> np.ndarray:
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    meta = np.ascontiguousarray(meta, dtype=np.float32)
    out = np.zeros(max(length, 1), dtype=np.float64)
    err = lib().qo_dequantize_segment(_ptr(codes), _ptr(meta), length, bucket, bits, _ptr(out),
                                      nthreads)
    if err:
        raise ValueError("nonzero padding bits in payload")
    return out[:length]


def encode_segment(codes, meta, length, bucket, bits) -> bytes:
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    meta = np.ascontiguousarray(meta, dtype=np.float32)
    out = np.zeros(message_size_bits(length, bucket, bits) // 8, dtype=np.uint8)
    n = lib().qo_encode_segment(_ptr(codes), _ptr(meta), length, bucket, bits, _ptr(out))
    return out[:n].tobytes()


def unpack(codes, length, bits) -> np.ndarray:
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    out = np.zeros(max(length, 1), dtype=np.uint32)
    lib().qo_unpack(_ptr(codes), length, bits, _ptr(out))
    return out[:length]


# -- learned levels (quantize.py:344-422) -----------------------------------------


def level_codes(u, levels) -> np.ndarray:
    """quantize_with_levels(u, LevelTable(levels), stochastic=False)."""
    q = np.ascontiguousarray(levels, dtype=np.float64)
    return np.array([lib().qo_level_code(float(x), _ptr(q), q.size) for x in np.atleast_1d(u)],
                    dtype=np.uint32)


def quantize_levels_segment(x, bucket, bits, levels):
    """bucketed_quantize(x, bucket, bits, "levels", levels=table) + packing.
    Returns (packed codes, meta float32[nb, 3], bad_index)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    q = np.ascontiguousarray(levels, dtype=np.float64)
    assert q.size == 1 << bits
    n = x.size
    codes = np.zeros(max(codes_bytes(n, bucket, bits), 1), dtype=np.uint8)
    meta = np.zeros((max(num_buckets(n, bucket), 1), 3), dtype=np.float32)
    bad = lib().qo_quantize_levels_segment(_ptr(x), n, bucket, bits, _ptr(q), _ptr(codes), _ptr(meta))
    return codes[: codes_bytes(n, bucket, bits)], meta[: num_buckets(n, bucket)], int(bad)


def dequantize_levels_segment(codes, meta, length, bucket, bits, levels) -> np.ndarray:
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    meta = np.ascontiguousarray(meta, dtype=np.float32)
    q = np.ascontiguousarray(levels, dtype=np.float64)
    out = np.zeros(max(length, 1), dtype=np.float64)
    if lib().qo_dequantize_levels_segment(_ptr(codes), _ptr(meta), length, bucket, bits, _ptr(q), _ptr(out)):
        raise ValueError("nonzero padding bits in payload")
    return out[:length]


def learn_levels(values, initial, lr=0.01) -> np.ndarray:
    """learn_levels(values, LevelTable(initial), lr).levels, including the
    distinct-count early return (quantize.py:366-397)."""
    v = np.ascontiguousarray(np.atleast_1d(values), dtype=np.float64)
    q = np.array(initial, dtype=np.float64)
    if v.size == 0:
        raise ValueError("cannot learn levels from an empty value set")
    if not np.all(np.isfinite(v)):
        raise ValueError("non-finite value")
    if np.unique(v).size < q.size:
        return q
    lib().qo_learn_levels(_ptr(v), v.size, _ptr(q), q.size, float(lr))
    return q


# -- protocol (sharded.py) -------------------------------------------------------


def shard_bounds(size: int, P: int):
    """sharded.py:193-200: contiguous partition, remainder to the last worker."""
    base = size // P
    b = [(p * base, (p + 1) * base) for p in range(P - 1)]
    b.append(((P - 1) * base, size))
    return b


def gather(full, P, bucket, bits, root, step, layer, phase, nthreads=1) -> np.ndarray:
    """Quantized all-gather of one flat layer (sharded.py:323-358, 530-550)."""
    full = np.asarray(full)
    parts = []
    for s, e in shard_bounds(full.size, P):
        if e == s:
            continue
        c, m, bad = quantize_segment(full[s:e], s, bucket, bits, SHIFT,
                                     (root, step, layer, phase, 0), nthreads)
        if bad >= 0:
            raise ValueError(f"non-finite bucket value at index {s + bad}")
        parts.append(dequantize_segment(c, m, e - s, bucket, bits, nthreads))
    return np.concatenate(parts) if parts else np.zeros(0)


def reduce_scatter(grads, bucket, bits, root, step, layer, nthreads=1):
    """Quantized reduce-scatter (sharded.py:375-433, 552-582): per destination
    q, sum the dequantized contributions of sources 0..P-1 in order, then /P."""
    P = len(grads)
    size = np.asarray(grads[0]).size
    out = []
    for q, (s, e) in enumerate(shard_bounds(size, P)):
        if e == s:
            out.append(np.zeros(0))
            continue
        acc = np.zeros(e - s)
        for p in range(P):
            seg = np.asarray(grads[p])[s:e]
            c, m, bad = quantize_segment(seg, s, bucket, bits, STOCHASTIC,
                                         (root, step, layer, PHASE_GRAD, p), nthreads)
            if bad >= 0:
                raise ValueError(f"non-finite bucket value at index {s + bad}")
            acc = acc + dequantize_segment(c, m, e - s, bucket, bits, nthreads)
        out.append(acc / P)
    return out
