"""Lattice-projected optimizer step fused with the reduce-scatter epilogue
(SURVEY §8(f) #4).

The reference's iteration (pkg/src/qsdp/optimizer.py:194-229, ``qsdp_step``;
PAPER.md:320-327) is

    y     = x - (eta / beta) * g
    x_new = d * round((y - r) / d) + r,      r = sample_shift(d, rng)

with ``np.round`` half-to-even.  In the sharded protocol ``g`` is the
reduce-scatter average of the P ranks' quantized gradients, so the step runs on
the owner's shard in the K4 epilogue: the fp64 average never leaves registers,
the iterate is read and written once.  The shift is the first draw of the
keyed stream ``bucket_rng(root, step, layer, PHASE_LATTICE, 0, 0)`` -- every rank
draws the same lattice without communication (the single-process reference
draws it from its sequential generator; ``qsdp_step(..., shift=r)`` with this r
reproduces our result bit-for-bit for fp64 iterates, tests/test_gpu_lattice.py).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import torch

from . import _lib
from .quantize import QuantSpec, SegmentKey, _DTYPE_CODE, _require_cuda, _stream

__all__ = ["PHASE_LATTICE", "LatticeStep", "shift_key", "dequant_accumulate_lattice"]

PHASE_LATTICE = 3


def shift_key(root_seed: int, step: int, layer: int) -> SegmentKey:
    """The key whose first draw gives the lattice shift of (step, layer)."""
    return SegmentKey(root_seed, step, layer, PHASE_LATTICE, 0)


@dataclass(frozen=True)
class LatticeStep:
    """``x <- d * rint((x - c*g - r)/d) + r`` with c = eta/beta, d = fine pitch."""

    lr_over_beta: float
    delta: float
    key: SegmentKey

    def __post_init__(self):
        if not self.delta > 0 or not math.isfinite(self.delta):
            raise ValueError(f"resolution must be > 0, got {self.delta}")

    def c(self, x_dtype: torch.dtype) -> _lib.Lattice:
        if x_dtype not in (torch.float32, torch.float64):
            raise ValueError("the iterate must be float32 or float64")
        return _lib.Lattice(float(self.lr_over_beta), float(self.delta), self.key.c(), _DTYPE_CODE[x_dtype])


def dequant_accumulate_lattice(sources, length: int, spec: QuantSpec, divisor: int, x: torch.Tensor,
                               step: LatticeStep, g_out: torch.Tensor | None = None):
    """K4 + lattice step: g = (0 + sum_p dequant(src_p)) / divisor (fp64, sources in
    order), then x (in place) moves to the shifted lattice.  ``g_out`` (optional)
    receives g.  Returns x."""
    _require_cuda(x, "iterate")
    if not x.is_contiguous() or x.numel() < length:
        raise ValueError("iterate must be contiguous and cover the segment")
    if len(sources) > 8:
        raise ValueError("at most 8 sources")
    n = len(sources)
    codes = (ctypes.c_void_p * n)(*[c.data_ptr() for c, _ in sources])
    metas = (ctypes.c_void_p * n)(*[m.data_ptr() for _, m in sources])
    lat = step.c(x.dtype)
    cfg = spec.cfg()
    gdt = g_out.dtype if g_out is not None else torch.float32
    with torch.cuda.device(x.device):
        _lib.check(_lib.lib().qsdp_dequant_accumulate_lattice(
            codes, metas, n, int(length), ctypes.byref(cfg), int(divisor),
            g_out.data_ptr() if g_out is not None else None, _DTYPE_CODE[gdt], x.data_ptr(), ctypes.byref(lat),
            _stream(x.device)))
    return x
