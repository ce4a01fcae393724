"""Bucketed QSDP quantizers on B200 -- tensor API plus the reference's
per-bucket API, both backed by the sm_100a kernels behind the C ABI.

Reference interface mirrored here (pkg/src/qsdp/quantize.py):

* ``quantize_bucket(values, bit_width, inner, rng)``       quantize.py:235-286
* ``bucketed_quantize(v, bucket, bit_width, inner, rng)``  quantize.py:289-313
* ``dequantize(block, mode, levels)``                      quantize.py:209-232
* inner mode ``"levels"`` (learned tables) routes to :mod:`.levels`
* ``QuantizedBlock`` / ``BucketSpec``                      quantize.py:64-127
* ``bucket_rng(root_seed, step, layer_idx, phase, worker, start)``
  (pkg/src/qsdp/sharded.py:235-240) returns a *key* the device generator
  reproduces bit-for-bit (numpy SeedSequence -> PCG64), instead of a host
  ``np.random.Generator``.

Tensor API (the hot path): :func:`quantize_segments`, :func:`dequantize_segments`,
:func:`dequant_accumulate` operate on CUDA tensors in the device layout of
include/qsdp_b200.h (packed codes + float32 ``[nb, 3]`` meta = shift, lo, hi).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

__all__ = [
    "QuantSpec", "SegmentKey", "BucketSpec", "QuantizedBlock", "KeyedBucketRNG", "bucket_rng", "philox_rng",
    "NOISE_MODES",
    "num_buckets", "codes_bytes", "message_size_bits", "quantize_segments", "quantize_segment",
    "dequantize_segments", "dequantize_segment", "dequant_accumulate", "quantize_bucket",
    "bucketed_quantize", "dequantize", "INNER_MODES", "advance_counter",
]

AFFINE_MODES = ("shift", "flip", "uniform_stochastic")
INNER_MODES = AFFINE_MODES + ("levels",)
_INNER_CODE = {"shift": _lib.INNER_SHIFT, "flip": _lib.INNER_STOCHASTIC,
               "uniform_stochastic": _lib.INNER_STOCHASTIC, "levels": _lib.INNER_LEVELS}
_DTYPE_CODE = {torch.float32: _lib.F32, torch.float64: _lib.F64, torch.bfloat16: _lib.BF16}
# the quantizers' noise (qsdp_noise): "pcg64" = bucket_rng's default_rng(SeedSequence(key)),
# "philox" = Generator(Philox(SeedSequence(key))) -- counter-based, same keys
NOISE_MODES = {"pcg64": 0, "philox": 1}


@dataclass(frozen=True)
class QuantSpec:
    """One tensor class of ``QuantConfig`` (sharded.py:76-93): width, bucket, inner mode."""

    bits: int = 8
    bucket: int = 1024
    inner: str = "shift"
    noise: str = "pcg64"

    def __post_init__(self):
        if not 1 <= self.bits <= 16:
            raise ValueError(f"bit_width must be in [1, 16], got {self.bits}")
        if self.bucket < 1:
            raise ValueError(f"bucket_size must be >= 1, got {self.bucket}")
        if self.inner not in _INNER_CODE:
            raise ValueError(f"unknown inner mode {self.inner!r}")
        if self.noise not in NOISE_MODES:
            raise ValueError(f"unknown noise mode {self.noise!r}")

    def cfg(self) -> _lib.QCfg:
        return _lib.QCfg(self.bits, self.bucket, _INNER_CODE[self.inner], NOISE_MODES[self.noise])


@dataclass(frozen=True)
class SegmentKey:
    """``bucket_rng`` key fields minus the bucket start (implicit per bucket)."""

    root_seed: int = 0
    step: int = 0
    layer: int = 0
    phase: int = 0
    worker: int = 0

    def c(self) -> _lib.Key:
        for v in (self.root_seed, self.step, self.layer, self.phase, self.worker):
            if v < 0 or v >= 1 << 64:
                raise ValueError("key fields must be non-negative 64-bit integers")
        return _lib.Key(self.root_seed, self.step, self.layer, self.phase, self.worker)


def num_buckets(length: int, bucket: int) -> int:
    return int(_lib.lib().qsdp_num_buckets(length, bucket))


def codes_bytes(length: int, spec: QuantSpec) -> int:
    cfg = spec.cfg()
    return int(_lib.lib().qsdp_codes_bytes(length, ctypes.byref(cfg)))


def message_size_bits(length: int, spec: QuantSpec) -> int:
    """Exact wire size of one encoded segment (wire.py:187-192)."""
    cfg = spec.cfg()
    return int(_lib.lib().qsdp_message_size_bits(length, ctypes.byref(cfg)))


def _stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _require_cuda(t: torch.Tensor, what: str) -> None:
    if not t.is_cuda:
        raise ValueError(f"{what} must be a CUDA tensor (no CPU fallback on the QSDP hot path)")


def _bad_to_error(bad: int, items) -> None:
    if bad == (1 << 64) - 1:
        return
    j, idx = bad >> 40, bad & ((1 << 40) - 1)
    x = items[j][0]
    v = float(x.view(-1)[idx].item())
    raise ValueError(f"non-finite bucket value at index {idx}: {v!r}")


def advance_counter(counter: torch.Tensor, delta: int = 1) -> None:
    """``counter += delta`` on the current stream via the library (graph-capturable)."""
    if counter.dtype != torch.int64 or not counter.is_cuda:
        raise ValueError("counter must be a CUDA int64 tensor")
    with torch.cuda.device(counter.device):
        _lib.check(_lib.lib().qsdp_counter_add(counter.data_ptr(), int(delta), _stream(counter.device)))


def quantize_segments(items, spec: QuantSpec, check_finite: bool = False, out=None, step_src=None):
    """Quantize several segments in one launch.

    ``items``: list of ``(x, global_start, SegmentKey)`` with ``x`` a contiguous
    1-D float32/float64 CUDA tensor; bucket j of a segment is keyed with start
    ``global_start + j*bucket`` (sharded.py:243-248).  Returns a list of
    ``(codes uint8[codes_bytes], meta float32[nb, 3])``.  With
    ``check_finite`` the call synchronises and raises ``ValueError`` naming the
    first non-finite element, like ``_check_finite`` (quantize.py:41-44).
    ``step_src`` (CUDA int64 scalar tensor): keys use ``step + step_src`` read on
    the device, so a captured CUDA graph replays with fresh noise per step.
    """
    if not items:
        return []
    dev = items[0][0].device
    dt = items[0][0].dtype
    if dt not in (torch.float32, torch.float64):
        raise ValueError("quantizer input must be float32 or float64")
    arr = (_lib.QItem * len(items))()
    outs = []
    for i, (x, gstart, key) in enumerate(items):
        _require_cuda(x, "input")
        if x.dtype != dt or x.device != dev:
            raise ValueError("all segments of one call share dtype and device")
        if not x.is_contiguous():
            raise ValueError("segments must be contiguous")
        n = x.numel()
        if out is not None:
            codes, meta = out[i]
        else:
            codes = torch.empty(max(codes_bytes(n, spec), 1), dtype=torch.uint8, device=dev)
            meta = torch.empty((max(num_buckets(n, spec.bucket), 1), 3), dtype=torch.float32, device=dev)
        arr[i].x = x.data_ptr()
        arr[i].seg = _lib.Segment(int(gstart), n)
        arr[i].key = key.c()
        arr[i].codes = codes.data_ptr()
        arr[i].meta = meta.data_ptr()
        outs.append((codes[: codes_bytes(n, spec)], meta[: num_buckets(n, spec.bucket)]))
    bad = None
    if check_finite:
        bad = torch.full((1,), -1, dtype=torch.int64, device=dev)  # all ones == UINT64_MAX
    cfg = spec.cfg()
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().qsdp_quantize_batch_dstep(
            arr, len(items), _DTYPE_CODE[dt], ctypes.byref(cfg),
            bad.data_ptr() if bad is not None else None,
            step_src.data_ptr() if step_src is not None else None, _stream(dev)))
    if bad is not None:
        _bad_to_error(int(bad.item()) & ((1 << 64) - 1), items)
    return outs


def quantize_segment(x, global_start: int, spec: QuantSpec, key: SegmentKey, check_finite=False):
    return quantize_segments([(x, global_start, key)], spec, check_finite=check_finite)[0]


def _ditems(jobs):
    arr = (_lib.DItem * len(jobs))()
    for i, (sources, length, out) in enumerate(jobs):
        if len(sources) > 8:
            raise ValueError("at most 8 sources per segment")
        for p, (codes, meta) in enumerate(sources):
            _require_cuda(codes, "codes")
            arr[i].codes[p] = codes.data_ptr()
            arr[i].meta[p] = meta.data_ptr()
        arr[i].nsrc = len(sources)
        arr[i].length = int(length)
        arr[i].out = out.data_ptr() if out is not None else None
    return arr


def dequantize_segments(jobs, spec: QuantSpec, dtype=torch.float32):
    """K3 over several segments: ``jobs`` = list of ``(codes, meta, length, out)``."""
    if not jobs:
        return
    dev = jobs[0][0].device
    for codes, meta, length, out in jobs:
        _require_cuda(out, "output")
        if out.dtype != dtype or out.numel() < length or not out.is_contiguous():
            raise ValueError("output must be a contiguous tensor of the requested dtype and length")
    arr = _ditems([([(c, m)], n, o) for c, m, n, o in jobs])
    cfg = spec.cfg()
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().qsdp_dequantize_batch(arr, len(jobs), ctypes.byref(cfg),
                                                    _DTYPE_CODE[dtype], _stream(dev)))


def dequantize_segment(codes, meta, length: int, spec: QuantSpec, dtype=torch.float32, out=None):
    if out is None:
        out = torch.empty(length, dtype=dtype, device=codes.device)
    dequantize_segments([(codes, meta, length, out)], spec, dtype)
    return out


def dequant_accumulate(sources, length: int, spec: QuantSpec, divisor: int, dtype=torch.float32,
                       out=None):
    """K4: ``(0 + sum_p dequant(src_p)) / divisor`` in fp64, sources in order."""
    if out is None:
        out = torch.empty(length, dtype=dtype, device=sources[0][0].device)
    dev = out.device
    arr = _ditems([(sources, length, out)])
    cfg = spec.cfg()
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().qsdp_dequant_accumulate_batch(arr, 1, ctypes.byref(cfg), int(divisor),
                                                            _DTYPE_CODE[dtype], _stream(dev)))
    return out


# ---------------------------------------------------------------------------
# The reference's per-bucket API (quantize.py), evaluated on the GPU.
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class BucketSpec:
    """Fixed-size bucketing with min-max normalisation (quantize.py:64-75)."""

    bucket_size: int = 1024
    normalization: str = "min_max"

    def __post_init__(self):
        if self.bucket_size < 1:
            raise ValueError(f"bucket_size must be >= 1, got {self.bucket_size}")
        if self.normalization != "min_max":
            raise ValueError(f"unknown normalization {self.normalization!r}")


class QuantizedBlock:
    """Same fields, invariants and equality as the reference's QuantizedBlock
    (quantize.py:78-127)."""

    def __init__(self, codes, shift, scale_lo, scale_hi, bit_width, length):
        self.codes = np.ascontiguousarray(codes, dtype=np.uint32)
        self.shift = float(shift)
        self.scale_lo = float(scale_lo)
        self.scale_hi = float(scale_hi)
        self.bit_width = int(bit_width)
        self.length = int(length)
        if self.length <= 0:
            raise ValueError("block length must be positive")
        if self.codes.shape != (self.length,):
            raise ValueError(f"expected {self.length} codes, got shape {self.codes.shape}")
        if not 1 <= self.bit_width <= 32:
            raise ValueError(f"bit_width must be in [1, 32], got {self.bit_width}")
        if self.codes.size and int(self.codes.max()) >= (1 << self.bit_width):
            raise ValueError(f"code out of range for bit_width {self.bit_width}")
        if not self.scale_lo <= self.scale_hi:
            raise ValueError("scale_lo must be <= scale_hi")

    @property
    def pitch(self) -> float:
        return (self.scale_hi - self.scale_lo) / ((1 << self.bit_width) - 1)

    def __eq__(self, other):
        if not isinstance(other, QuantizedBlock):
            return NotImplemented
        return (self.length == other.length and self.bit_width == other.bit_width
                and self.shift == other.shift and self.scale_lo == other.scale_lo
                and self.scale_hi == other.scale_hi and np.array_equal(self.codes, other.codes))

    def __repr__(self):
        return (f"QuantizedBlock(length={self.length}, bit_width={self.bit_width}, shift={self.shift!r}, "
                f"scale_lo={self.scale_lo!r}, scale_hi={self.scale_hi!r})")


class KeyedBucketRNG:
    """What ``bucket_rng`` returns here: the key of one quantization event.
    The device regenerates numpy's SeedSequence(key) -> PCG64 stream from it
    (``noise="philox"``: the Philox4x64-10 stream of the same SeedSequence)."""

    __slots__ = ("key", "start", "noise")

    def __init__(self, root_seed, step, layer_idx, phase, worker, start, noise="pcg64"):
        self.key = SegmentKey(int(root_seed), int(step), int(layer_idx), int(phase), int(worker))
        self.start = int(start)
        self.noise = noise


def bucket_rng(root_seed: int, step: int, layer_idx: int, phase: int, worker: int,
               start: int) -> KeyedBucketRNG:
    """Deterministic generator key for one quantization event (sharded.py:235-240)."""
    for v in (root_seed, step, layer_idx, phase, worker, start):
        if int(v) < 0:
            raise ValueError("expected non-negative integer key fields")
    return KeyedBucketRNG(root_seed, step, layer_idx, phase, worker, start)


def philox_rng(root_seed: int, step: int, layer_idx: int, phase: int, worker: int,
               start: int) -> KeyedBucketRNG:
    """The counter-based generator of the same key:
    ``np.random.Generator(np.random.Philox(SeedSequence((root, step, layer, phase, worker, start))))``
    -- a generator the reference's ``quantize_bucket`` accepts (quantize.py:235-241)."""
    for v in (root_seed, step, layer_idx, phase, worker, start):
        if int(v) < 0:
            raise ValueError("expected non-negative integer key fields")
    return KeyedBucketRNG(root_seed, step, layer_idx, phase, worker, start, noise="philox")


def _unpack(packed: np.ndarray, n: int, bits: int) -> np.ndarray:
    bitsarr = np.unpackbits(packed, bitorder="little")[: n * bits].reshape(n, bits).astype(np.uint64)
    return (bitsarr @ (np.uint64(1) << np.arange(bits, dtype=np.uint64))).astype(np.uint32)


def _pack(codes: np.ndarray, bits: int) -> np.ndarray:
    b = ((codes.astype(np.uint32)[:, None] >> np.arange(bits, dtype=np.uint32)) & 1).astype(np.uint8)
    return np.packbits(b.ravel(), bitorder="little")


def _blocks_from_device(codes_t, meta_t, n, bucket, bits):
    packed = codes_t.cpu().numpy()
    meta = meta_t.cpu().numpy().astype(np.float64)
    pbs = (bucket * bits + 7) // 8
    blocks = []
    for j in range(meta.shape[0]):
        m = min(bucket, n - j * bucket)
        pb = (m * bits + 7) // 8
        c = _unpack(packed[j * pbs: j * pbs + pb], m, bits)
        blocks.append(QuantizedBlock(c, meta[j, 0], meta[j, 1], meta[j, 2], bits, m))
    return blocks


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("the QSDP B200 path needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


_PCG_M = 0x2360ED051FC65DA44385DF649FCCF645
_MASK128 = (1 << 128) - 1


def _pcg_advance_coeffs(k: int):
    """(A_k, G_k) with state_k = A_k * state + G_k * inc (mod 2^128): numpy PCG64 after k draws."""
    am, ap, cm, cp = 1, 0, _PCG_M, 1
    while k:
        if k & 1:
            am = am * cm & _MASK128
            ap = (ap * cm + cp) & _MASK128
        cp = (cm + 1) * cp & _MASK128
        cm = cm * cm & _MASK128
        k >>= 1
    return am, ap


def _shared_stream_blocks(v: np.ndarray, bucket: int, bit_width: int, inner: str, rng) -> list:
    """bucketed_quantize with ONE numpy Generator consumed in bucket order (quantize.py:289-313):
    a non-degenerate bucket draws 1 (shift) or n (stochastic) outputs, a degenerate bucket none
    (quantize.py:256-264).  The prefix sum of draws gives every bucket's starting PCG64 state;
    the device quantizes all buckets at once from those states, and ``rng`` is advanced past
    the draws, exactly where the reference leaves it."""
    bg = rng.bit_generator
    if not isinstance(bg, np.random.PCG64):
        raise TypeError("a shared generator must be numpy PCG64 (np.random.default_rng): the device replays its stream")
    if not 1 <= bit_width <= 16:
        raise ValueError(f"bit_width must be in [1, 16], got {bit_width}")
    n = v.size
    starts = np.arange(0, n, bucket)
    lens = np.minimum(bucket, n - starts)
    bad = np.flatnonzero(~np.isfinite(v))
    nb = starts.size if bad.size == 0 else int(bad[0] // bucket)  # buckets quantized before a raise
    lo = np.minimum.reduceat(v, starts).astype(np.float32) if n else np.zeros(0, np.float32)
    hi = np.maximum.reduceat(v, starts).astype(np.float32) if n else np.zeros(0, np.float32)
    draws = np.where(lo == hi, 0, 1 if inner == "shift" else lens).astype(np.int64)
    st = bg.state["state"]
    state, inc = int(st["state"]), int(st["inc"])
    common = int(draws.max()) if draws.size else 0
    a_c, g_c = _pcg_advance_coeffs(common)
    words = np.zeros((max(nb, 1), 4), dtype=np.uint64)
    cur = state
    for j in range(nb):
        words[j] = (cur & 0xFFFFFFFFFFFFFFFF, cur >> 64, inc & 0xFFFFFFFFFFFFFFFF, inc >> 64)
        d = int(draws[j])
        if d:
            a, g = (a_c, g_c) if d == common else _pcg_advance_coeffs(d)
            cur = (a * cur + g * inc) & _MASK128
    if bad.size:  # the reference consumed the earlier buckets' draws, then raised in _check_finite
        bg.advance(int(draws[:nb].sum()))
        i = int(bad[0])
        raise ValueError(f"non-finite bucket value at index {i - nb * bucket}: {v[i]!r}")
    dev = _device()
    spec = QuantSpec(bit_width, bucket, inner)
    cfg = spec.cfg()
    x = torch.from_numpy(np.ascontiguousarray(v)).to(dev)
    states = torch.from_numpy(words.view(np.int64)).to(dev)
    codes = torch.empty(max(codes_bytes(n, spec), 1), dtype=torch.uint8, device=dev)
    meta = torch.empty((max(num_buckets(n, bucket), 1), 3), dtype=torch.float32, device=dev)
    scratch = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().qsdp_quantize_stream(x.data_ptr(), _lib.F64, n, ctypes.byref(cfg), states.data_ptr(),
                                                   codes.data_ptr(), meta.data_ptr(), scratch.data_ptr(),
                                                   _stream(dev)))
    blocks = _blocks_from_device(codes, meta, n, bucket, bit_width)
    bg.advance(int(draws.sum()))
    return blocks


def quantize_bucket(values, bit_width: int, inner: str, rng, levels=None) -> QuantizedBlock:
    """Min-max normalise one bucket and quantize it on the GPU (quantize.py:235-286).

    ``rng``: a ``bucket_rng`` / ``philox_rng`` key (the device regenerates the keyed stream),
    or a numpy PCG64 Generator, whose stream the device continues (and advances)."""
    v = np.asarray(values, dtype=float)
    if v.size == 0:
        raise ValueError("cannot quantize an empty bucket")
    if inner not in INNER_MODES:
        raise ValueError(f"unknown inner mode {inner!r}")
    if inner == "levels":  # no draws: rng is not consulted (quantize.py:275-279)
        return _levels_blocks(v, v.size, bit_width, levels)[0]
    if isinstance(rng, np.random.Generator):
        return _shared_stream_blocks(v, v.size, bit_width, inner, rng)[0]
    if not isinstance(rng, KeyedBucketRNG):
        raise TypeError("rng must come from bucket_rng(...): the device reproduces keyed streams")
    spec = QuantSpec(bit_width, v.size, inner, rng.noise)
    x = torch.from_numpy(np.ascontiguousarray(v)).to(_device())
    codes, meta = quantize_segment(x, rng.start, spec, rng.key, check_finite=True)
    return _blocks_from_device(codes, meta, v.size, v.size, bit_width)[0]


def bucketed_quantize(v, bucket: BucketSpec, bit_width: int, inner: str = "shift", rng=None,
                      levels=None) -> list:
    """Split into buckets and quantize each (quantize.py:289-313).

    ``rng`` = a numpy PCG64 Generator (or None: ``np.random.default_rng()``, as the
    reference): ONE stream shared by the buckets in order, replayed on the device and
    advanced like the reference's; or a ``bucket_rng(...)`` / ``philox_rng(...)`` key:
    bucket j keyed with ``start + j*bucket_size`` exactly like ``_segment_blocks``
    (sharded.py:243-248).
    """
    v = np.atleast_1d(np.asarray(v, dtype=float))
    if v.size == 0:
        raise ValueError("cannot quantize an empty vector")
    if not 1 <= bit_width <= 16:
        raise ValueError(f"bit_width must be in [1, 16], got {bit_width}")
    if inner == "levels":
        return _levels_blocks(v, bucket.bucket_size, bit_width, levels)
    if inner not in INNER_MODES:
        raise ValueError(f"unknown inner mode {inner!r}")
    if rng is None:
        rng = np.random.default_rng()
    if isinstance(rng, np.random.Generator):
        return _shared_stream_blocks(v, bucket.bucket_size, bit_width, inner, rng)
    if not isinstance(rng, KeyedBucketRNG):
        raise TypeError("rng must be a numpy PCG64 Generator or come from bucket_rng(...)")
    spec = QuantSpec(bit_width, bucket.bucket_size, inner, rng.noise)
    x = torch.from_numpy(np.ascontiguousarray(v)).to(_device())
    codes, meta = quantize_segment(x, rng.start, spec, rng.key, check_finite=True)
    return _blocks_from_device(codes, meta, v.size, bucket.bucket_size, bit_width)


def dequantize(block: QuantizedBlock, mode: str = "shift", levels=None) -> np.ndarray:
    """Reconstruct a block on the GPU: (lo + code*pitch) + shift in fp64 (quantize.py:209-232)."""
    if mode not in INNER_MODES:
        raise ValueError(f"unknown mode {mode!r}")
    codes = np.asarray(block.codes)
    if codes.size and int(codes.max()) >= (1 << block.bit_width):
        raise ValueError(f"corrupted code >= 2**{block.bit_width} cannot be decoded")
    if mode == "levels":
        if levels is None:
            raise ValueError("mode 'levels' requires a LevelTable")
        if levels.levels.size != (1 << block.bit_width):
            raise ValueError("level table size does not match bit_width")
    dev = _device()
    spec = QuantSpec(block.bit_width, block.length, "levels" if mode == "levels" else "shift")
    packed = torch.from_numpy(_pack(codes, block.bit_width)).to(dev)
    meta = torch.tensor([[block.shift, block.scale_lo, block.scale_hi]], dtype=torch.float32, device=dev)
    if float(np.float32(block.shift)) != block.shift or float(np.float32(block.scale_lo)) != block.scale_lo \
            or float(np.float32(block.scale_hi)) != block.scale_hi:
        raise ValueError("device dequantize takes float32-exact block metadata (the wire format's)")
    if mode == "levels":
        from .levels import dequantize_levels
        out = dequantize_levels(packed, meta, block.length, spec, levels, dtype=torch.float64)
    else:
        out = dequantize_segment(packed, meta, block.length, spec, dtype=torch.float64)
    return out.cpu().numpy()


def _levels_blocks(v: np.ndarray, bucket: int, bit_width: int, levels) -> list:
    """inner="levels" over consecutive buckets on the GPU (quantize.py:275-279, 400-416)."""
    if levels is None:
        raise ValueError("inner 'levels' requires a LevelTable")
    from .levels import quantize_levels
    if not 1 <= bit_width <= 16:
        raise ValueError(f"bit_width must be in [1, 16], got {bit_width}")
    if levels.levels.size > (1 << bit_width):
        raise ValueError(f"code out of range for bit_width {bit_width}")
    spec = QuantSpec(bit_width, bucket, "levels")
    x = torch.from_numpy(np.ascontiguousarray(v)).to(_device())
    codes, meta = quantize_levels(x, spec, levels, check_finite=True)
    return _blocks_from_device(codes, meta, v.size, bucket, bit_width)
