"""Learned quantization levels on B200.

Mirrors the reference's non-uniform codebook API (pkg/src/qsdp/quantize.py):

* ``LevelTable``                                        quantize.py:344-363
* ``learn_levels(values, initial, learning_rate)``      quantize.py:366-397
* ``quantize_with_levels(v, table, stochastic=False)``  quantize.py:400-422
* ``quantize_bucket(..., "levels", levels=table)``      quantize.py:235-286
  and ``dequantize(block, "levels", table)``            quantize.py:225-231
  (routed here from :mod:`.quantize`)

Quantize / dequantize / learn run as sm_100a kernels behind the C ABI
(``qsdp_quantize_levels*``, ``qsdp_dequantize_levels*``, ``qsdp_learn_levels``);
results are bit-identical to the reference (tests/test_gpu_levels.py).  The
level table itself is a tiny host array (<= 2^16 doubles) uploaded once per
table, as the reference keeps it on the host.
"""

from __future__ import annotations

import ctypes
import warnings

import numpy as np
import torch

from . import _lib
from .quantize import QuantSpec, _DTYPE_CODE, _require_cuda, _stream, codes_bytes, num_buckets

__all__ = ["LevelTable", "learn_levels", "quantize_with_levels", "quantize_levels", "quantize_levels_segments",
           "dequantize_levels", "learn_weight_levels"]


class LevelTable:
    """Strictly increasing quantization levels; count is a power of two (quantize.py:344-363)."""

    def __init__(self, levels):
        self.levels = np.ascontiguousarray(levels, dtype=float)
        n = self.levels.size
        if n < 1 or (n & (n - 1)) != 0:
            raise ValueError(f"level count must be a power of two, got {n}")
        if n > 1 and not np.all(np.diff(self.levels) > 0):
            raise ValueError("levels must be strictly increasing")
        self._dev = {}

    @property
    def bit_width(self) -> int:
        return int(self.levels.size).bit_length() - 1

    @classmethod
    def uniform(cls, bit_width: int, lo: float = 0.0, hi: float = 1.0) -> "LevelTable":
        return cls(np.linspace(lo, hi, 1 << bit_width))

    def device(self, dev) -> torch.Tensor:
        """The table as a float64 tensor on ``dev`` (uploaded once)."""
        dev = torch.device(dev)
        t = self._dev.get(dev)
        if t is None:
            t = torch.from_numpy(self.levels.copy()).to(dev)
            self._dev[dev] = t
        return t

    def __repr__(self):
        return f"LevelTable(levels={self.levels!r})"


def _as_device_f64(values, dev=None) -> torch.Tensor:
    if isinstance(values, torch.Tensor):
        _require_cuda(values, "values")
        return values.reshape(-1).to(torch.float64).contiguous()
    v = np.atleast_1d(np.asarray(values, dtype=float))
    if dev is None:
        if not torch.cuda.is_available():
            raise RuntimeError("the QSDP B200 path needs a CUDA device (no CPU fallback)")
        dev = torch.device("cuda", torch.cuda.current_device())
    return torch.from_numpy(np.ascontiguousarray(v)).to(dev)


def _first_nonfinite(v: torch.Tensor):
    bad = torch.nonzero(~torch.isfinite(v))
    if bad.numel():
        i = int(bad[0, 0])
        return i, float(v[i])
    return None


def learn_levels(values, initial: LevelTable, learning_rate: float = 0.01) -> LevelTable:
    """One pass of gradient descent on the level locations (quantize.py:366-397),
    on the GPU: values are visited in order by one warp (the update is
    sequential), the table lives in shared memory."""
    v = _as_device_f64(values)
    if v.numel() == 0:
        raise ValueError("cannot learn levels from an empty value set")
    bad = _first_nonfinite(v)
    if bad is not None:
        raise ValueError(f"non-finite value at index {bad[0]}: {bad[1]!r}")
    q0 = initial.levels
    if q0.size > 4096:
        raise ValueError("learn_levels on the device supports tables of up to 2**12 levels")
    if torch.unique(v).numel() < q0.size:
        warnings.warn("fewer distinct values than levels; returning the initial table", RuntimeWarning)
        return LevelTable(q0.copy())
    q = torch.from_numpy(q0.copy()).to(v.device)
    with torch.cuda.device(v.device):
        _lib.check(_lib.lib().qsdp_learn_levels(v.data_ptr(), v.numel(), q.data_ptr(), q.numel(),
                                                float(learning_rate), _stream(v.device)))
    return LevelTable(q.cpu().numpy())


def quantize_with_levels(v, table: LevelTable, stochastic: bool = False, rng=None):
    """Map values to level indices, clamping outside the table's span (quantize.py:400-422).
    Returns codes in the input's container type (numpy uint32 for array-likes, int64 CUDA
    tensor for tensors).  ``stochastic=True`` rounds to the bracketing levels with the draws
    of ``rng`` (a numpy PCG64 Generator, continued on the device and advanced by v.size
    draws, as the reference's rng.random(v.size))."""
    if stochastic:
        if rng is None:
            raise ValueError("stochastic mode requires an rng")
        return _levels_stochastic(v, table, rng)
    is_t = isinstance(v, torch.Tensor)
    x = _as_device_f64(v)
    q = table.device(x.device)
    if q.numel() == 1:
        codes = torch.zeros(x.numel(), dtype=torch.int64, device=x.device)
    else:
        x = torch.clamp(x, q[0], q[-1])
        mids = (q[:-1] + q[1:]) / 2
        codes = torch.searchsorted(mids, x, side="left")
    return codes if is_t else codes.cpu().numpy().astype(np.uint32)


def _levels_stochastic(v, table: LevelTable, rng):
    is_t = isinstance(v, torch.Tensor)
    x = _as_device_f64(v)
    n = x.numel()
    q = table.device(x.device)
    if q.numel() == 1:  # the reference returns before drawing
        codes = torch.zeros(n, dtype=torch.int64, device=x.device)
        return codes if is_t else codes.cpu().numpy().astype(np.uint32)
    bg = rng.bit_generator
    if not isinstance(bg, np.random.PCG64):
        raise TypeError("stochastic levels replay a numpy PCG64 Generator (np.random.default_rng)")
    st = bg.state["state"]
    state, inc = int(st["state"]), int(st["inc"])
    words = (ctypes.c_uint64 * 4)(state & 0xFFFFFFFFFFFFFFFF, state >> 64, inc & 0xFFFFFFFFFFFFFFFF, inc >> 64)
    out = torch.empty(max(n, 1), dtype=torch.int32, device=x.device)
    with torch.cuda.device(x.device):
        _lib.check(_lib.lib().qsdp_levels_stochastic(x.data_ptr(), n, q.data_ptr(), q.numel(), words, out.data_ptr(),
                                                     _stream(x.device)))
    bg.advance(n)
    codes = out[:n].to(torch.int64)
    return codes if is_t else codes.cpu().numpy().astype(np.uint32)


def _levels_spec(spec: QuantSpec) -> QuantSpec:
    if spec.inner != "levels":
        raise ValueError("levels entry points take a QuantSpec with inner='levels'")
    return spec


def quantize_levels_segments(xs, spec: QuantSpec, table: LevelTable, check_finite: bool = False, out=None):
    """Bucketed levels quantization of several segments in one launch.

    ``xs``: contiguous 1-D float32/float64 CUDA tensors.  Returns a list of
    ``(codes uint8[codes_bytes], meta float32[nb, 3])`` with meta shift 0.
    """
    _levels_spec(spec)
    if not xs:
        return []
    dev, dt = xs[0].device, xs[0].dtype
    if dt not in (torch.float32, torch.float64):
        raise ValueError("quantizer input must be float32 or float64")
    arr = (_lib.QItem * len(xs))()
    outs = []
    for i, x in enumerate(xs):
        _require_cuda(x, "input")
        if x.dtype != dt or x.device != dev or not x.is_contiguous():
            raise ValueError("segments must be contiguous and share dtype and device")
        n = x.numel()
        if out is not None:
            codes, meta = out[i]
        else:
            codes = torch.empty(max(codes_bytes(n, spec), 1), dtype=torch.uint8, device=dev)
            meta = torch.empty((max(num_buckets(n, spec.bucket), 1), 3), dtype=torch.float32, device=dev)
        arr[i].x = x.data_ptr()
        arr[i].seg = _lib.Segment(0, n)
        arr[i].codes = codes.data_ptr()
        arr[i].meta = meta.data_ptr()
        outs.append((codes[: codes_bytes(n, spec)], meta[: num_buckets(n, spec.bucket)]))
    q = table.device(dev)
    bad = torch.full((1,), -1, dtype=torch.int64, device=dev) if check_finite else None
    cfg = spec.cfg()
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().qsdp_quantize_levels_batch(
            arr, len(xs), _DTYPE_CODE[dt], ctypes.byref(cfg), q.data_ptr(), q.numel(),
            bad.data_ptr() if bad is not None else None, _stream(dev)))
    if bad is not None:
        b = int(bad.item()) & ((1 << 64) - 1)
        if b != (1 << 64) - 1:
            j, idx = b >> 40, b & ((1 << 40) - 1)
            raise ValueError(f"non-finite bucket value at index {idx}: {float(xs[j][idx])!r}")
    return outs


def quantize_levels(x, spec: QuantSpec, table: LevelTable, check_finite: bool = False):
    return quantize_levels_segments([x], spec, table, check_finite)[0]


def dequantize_levels(codes, meta, length: int, spec: QuantSpec, table: LevelTable, dtype=torch.float64,
                      out=None):
    """``lo + levels[code] * (hi - lo)`` per bucket (quantize.py:225-231)."""
    _levels_spec(spec)
    _require_cuda(codes, "codes")
    dev = codes.device
    if out is None:
        out = torch.empty(length, dtype=dtype, device=dev)
    if out.dtype != dtype or out.numel() < length or not out.is_contiguous():
        raise ValueError("output must be a contiguous tensor of the requested dtype and length")
    q = table.device(dev)
    cfg = spec.cfg()
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().qsdp_dequantize_levels(codes.data_ptr(), meta.data_ptr(), int(length),
                                                     ctypes.byref(cfg), q.data_ptr(), q.numel(),
                                                     out.data_ptr(), _DTYPE_CODE[dtype], _stream(dev)))
    return out


def _normalize_buckets(x: torch.Tensor, bucket_size: int):
    """Bucket-wise fp64 min-max normalisation as in experiments.py:418-426:
    returns (u, lo, span) per element, u = (x - lo) / span (0 where span == 0)."""
    x = x.reshape(-1).to(torch.float64)
    n = x.numel()
    nb = -(-n // bucket_size)
    pad = nb * bucket_size - n
    xp = torch.cat([x, x[-1:].expand(pad)]) if pad else x  # padding repeats a member: min/max unchanged
    tiles = xp.view(nb, bucket_size)
    lo = tiles.amin(dim=1, keepdim=True)
    span = tiles.amax(dim=1, keepdim=True) - lo
    u = torch.where(span > 0, (tiles - lo) / torch.where(span > 0, span, torch.ones_like(span)),
                    torch.zeros_like(tiles))
    lo_e = lo.expand(nb, bucket_size).reshape(-1)[:n]
    span_e = span.expand(nb, bucket_size).reshape(-1)[:n]
    return u.reshape(-1)[:n].contiguous(), lo_e, span_e


def learn_weight_levels(tensors, bit_width: int, bucket_size: int = 1024, learning_rate: float = 0.01,
                        passes: int = 1, max_values: int = 1 << 18, seed: int = 0) -> LevelTable:
    """A weight level table for the levels all-gather: the bucket-normalised
    values of ``tensors`` (a strided sample of at most ``max_values``), then
    ``passes`` learn_levels passes from the uniform table (Alg. 2)."""
    us = [_normalize_buckets(t.detach().reshape(-1), bucket_size)[0] for t in tensors if t.numel()]
    u = torch.cat(us)
    if u.numel() > max_values:
        g = torch.Generator(device=u.device).manual_seed(seed)
        u = u[torch.randperm(u.numel(), generator=g, device=u.device)[:max_values]]
    table = LevelTable.uniform(bit_width)
    for _ in range(passes):
        table = learn_levels(u, table, learning_rate)
    return table
