"""Byte-exact QSDP wire messages on B200.

Mirrors pkg/src/qsdp/wire.py:

* ``encode(blocks) -> bytes`` / ``decode(data) -> list[QuantizedBlock]`` /
  ``message_size_bits(blocks)`` (wire.py:108-192) with the same validation,
  exception types and error precedence (``WireError`` > ``EncodeError`` /
  ``DecodeError`` > ``TruncatedMessageError`` / ``UnsupportedVersionError`` /
  ``CodeRangeError``, wire.py:54-75);
* the device codec the reference does not have: :func:`encode_segment` turns a
  quantized segment in the device layout (packed codes + float32 [nb, 3] meta,
  what the quantizers and collectives produce) into the message on the GPU, and
  :func:`decode_segment` turns a message in device memory back into the device
  layout -- for checkpointing quantized state or shipping it across nodes.

The message bytes are identical to the reference's encoder's for the same blocks
(tests/test_gpu_wire.py against tests/golden).  The codec carries any width a
QuantizedBlock may hold (1..32); the quantizers produce 1..16.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import (CodeRangeError, DecodeError, EncodeError, TruncatedMessageError, UnsupportedVersionError,
                   WireError)
from .quantize import QuantizedBlock, QuantSpec, _device, _require_cuda, _stream

__all__ = ["WIRE_VERSION", "HEADER_BITS", "BLOCK_META_BITS", "encode", "decode", "message_size_bits",
           "encode_segment", "decode_segment", "DecodedSegment", "WireError", "EncodeError", "DecodeError",
           "TruncatedMessageError", "UnsupportedVersionError", "CodeRangeError", "pack_codes", "unpack_codes"]

WIRE_VERSION = 1
HEADER_BITS = 14 * 8
BLOCK_META_BITS = 12 * 8


def _payload_bytes(length: int, bit_width: int) -> int:
    return (length * bit_width + 7) // 8


def _cfg(bits: int, bucket: int) -> _lib.QCfg:
    return _lib.QCfg(int(bits), int(bucket), _lib.INNER_SHIFT, 0)


def _codes_bytes(length: int, bits: int, bucket: int) -> int:
    if length <= 0:
        return 0
    nb = -(-length // bucket)
    return (nb - 1) * _payload_bytes(bucket, bits) + _payload_bytes(length - (nb - 1) * bucket, bits)


def _msg_bytes(length: int, bits: int, bucket: int) -> int:
    return 14 + (12 * -(-length // bucket) + _codes_bytes(length, bits, bucket) if length > 0 else 0)


def pack_codes(codes: torch.Tensor, bits: int, bucket: int) -> torch.Tensor:
    """uint32 (int64/int32 accepted) CUDA codes -> the packed device layout."""
    _require_cuda(codes, "codes")
    c = codes.to(torch.int64).to(torch.int32).contiguous()  # uint32 bit patterns
    n = c.numel()
    nbytes = _codes_bytes(n, bits, bucket)
    out = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=c.device)
    cfg = _cfg(bits, bucket)
    with torch.cuda.device(c.device):
        _lib.check(_lib.lib().qsdp_pack_codes(c.data_ptr(), n, ctypes.byref(cfg), out.data_ptr(), _stream(c.device)))
    return out[:nbytes]


def unpack_codes(packed: torch.Tensor, length: int, bits: int, bucket: int) -> torch.Tensor:
    """The packed device layout -> int32 CUDA codes (one per element)."""
    _require_cuda(packed, "packed")
    out = torch.empty(max(length, 1), dtype=torch.int32, device=packed.device)
    cfg = _cfg(bits, bucket)
    with torch.cuda.device(packed.device):
        _lib.check(_lib.lib().qsdp_unpack_codes(packed.data_ptr(), int(length), ctypes.byref(cfg), out.data_ptr(),
                                                _stream(packed.device)))
    return out[:length]


def encode_segment(codes: torch.Tensor, meta: torch.Tensor, length: int, spec,
                   out: torch.Tensor | None = None) -> torch.Tensor:
    """Device layout -> message (uint8 CUDA tensor of message_size_bits/8 bytes).
    ``spec``: a QuantSpec, or ``(bits, bucket)`` for widths above 16."""
    _require_cuda(codes, "codes")
    _require_cuda(meta, "meta")
    bits, bucket = (spec.bits, spec.bucket) if isinstance(spec, QuantSpec) else (int(spec[0]), int(spec[1]))
    nbytes = _msg_bytes(int(length), bits, bucket)
    if out is None:
        out = torch.empty(nbytes, dtype=torch.uint8, device=codes.device)
    cfg = _cfg(bits, bucket)
    with torch.cuda.device(codes.device):
        _lib.check(_lib.lib().qsdp_wire_encode_device(codes.data_ptr(), meta.data_ptr(), int(length),
                                                      ctypes.byref(cfg), out.data_ptr(), out.numel(),
                                                      _stream(codes.device)))
    return out[:nbytes]


@dataclass
class DecodedSegment:
    codes: torch.Tensor  # packed device layout
    meta: torch.Tensor   # float32 [nb, 3]: shift, scale_lo, scale_hi
    length: int
    bits: int
    bucket: int


def decode_segment(msg: torch.Tensor) -> DecodedSegment:
    """Message in device memory -> device layout, raising exactly what the
    reference ``decode`` raises for the same bytes (wire.py:134-184)."""
    _require_cuda(msg, "message")
    if msg.dtype != torch.uint8 or msg.dim() != 1:
        raise ValueError("message must be a 1-D uint8 tensor")
    n = msg.numel()
    hdr = msg[: min(14, n)].cpu().numpy()
    info = _lib.WireInfo()
    _lib.check(_lib.lib().qsdp_wire_parse(hdr.ctypes.data if n else None, n, ctypes.byref(info)))
    dev = msg.device
    if info.blocks == 0:
        return DecodedSegment(torch.empty(0, dtype=torch.uint8, device=dev),
                              torch.empty((0, 3), dtype=torch.float32, device=dev), 0, info.bits, info.bucket)
    L, bits, bucket = int(info.total_length), int(info.bits), int(info.bucket)
    nb = -(-L // bucket)
    codes = torch.zeros(max(_codes_bytes(L, bits, bucket), 1), dtype=torch.uint8, device=dev)
    meta = torch.zeros((max(nb, 1), 3), dtype=torch.float32, device=dev)
    err = torch.full((2,), -1, dtype=torch.int64, device=dev)
    msgc = msg.contiguous()
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().qsdp_wire_decode_device(msgc.data_ptr(), ctypes.byref(info), codes.data_ptr(),
                                                      meta.data_ptr(), err.data_ptr(), _stream(dev)))
    e = [int(v) & ((1 << 64) - 1) for v in err.cpu().tolist()]
    none = (1 << 64) - 1
    t = int(info.complete_blocks)  # first block not wholly present
    first = min(e[0], e[1])
    if first != none and first < t:  # block order: padding check, then QuantizedBlock's scale check
        if e[0] == first:
            raise DecodeError("nonzero padding bits in payload")
        raise ValueError("scale_lo must be <= scale_hi")
    if t < info.blocks:
        blk = 12 + _payload_bytes(int(info.bucket), info.bits)
        if 14 + t * blk + 12 > n:
            raise TruncatedMessageError(f"block {t} metadata truncated")
        raise TruncatedMessageError(f"block {t} payload truncated")
    if n != info.expected_bytes:
        raise DecodeError(f"{n - info.expected_bytes} unexpected trailing bytes")
    return DecodedSegment(codes[: _codes_bytes(L, bits, bucket)], meta[:nb], L, bits, bucket)


def decode_kernels(msgs):
    """A callable launching only the decode kernels of well-formed ``msgs``
    (headers parsed once up front): for timing / CUDA-graph capture."""
    jobs = []
    for m in msgs:
        n = m.numel()
        hdr = m[:14].cpu().numpy()
        info = _lib.WireInfo()
        _lib.check(_lib.lib().qsdp_wire_parse(hdr.ctypes.data, n, ctypes.byref(info)))
        L, bits, bucket = int(info.total_length), int(info.bits), int(info.bucket)
        codes = torch.empty(max(_codes_bytes(L, bits, bucket), 1), dtype=torch.uint8, device=m.device)
        meta = torch.empty((max(-(-L // bucket), 1), 3), dtype=torch.float32, device=m.device)
        err = torch.full((2,), -1, dtype=torch.int64, device=m.device)
        jobs.append((m, info, codes, meta, err))

    def run():
        for m, info, codes, meta, err in jobs:
            _lib.check(_lib.lib().qsdp_wire_decode_device(m.data_ptr(), ctypes.byref(info), codes.data_ptr(),
                                                          meta.data_ptr(), err.data_ptr(), _stream(m.device)))
    return run


# ---------------------------------------------------------------------------
# The reference's host-object API (blocks in host memory), on the device codec.
# ---------------------------------------------------------------------------


def message_size_bits(blocks) -> int:
    """Exact encoded size in bits, metadata and per-block padding included (wire.py:187-192)."""
    size = HEADER_BITS
    for b in blocks:
        size += BLOCK_META_BITS + 8 * _payload_bytes(b.length, b.bit_width)
    return size


def encode(blocks) -> bytes:
    """Serialize a canonical (bucket-shaped) block list (wire.py:108-131)."""
    if not blocks:
        return bytes([WIRE_VERSION]) + bytes(13)
    bit_width = blocks[0].bit_width
    bucket_size = blocks[0].length
    total = 0
    for i, b in enumerate(blocks):
        if b.bit_width != bit_width:
            raise EncodeError(f"mixed bit_width: block 0 has {bit_width}, block {i} has {b.bit_width}")
        last = i == len(blocks) - 1
        if not last and b.length != bucket_size:
            raise EncodeError("only the final block may be shorter than the bucket")
        if last and b.length > bucket_size:
            raise EncodeError("final block exceeds the bucket size")
        total += b.length
    for b in blocks:
        for name in ("shift", "scale_lo", "scale_hi"):
            val = getattr(b, name)
            if float(np.float32(val)) != val:
                raise EncodeError(f"block {name}={val!r} is not float32-exact; the wire carries "
                                  "f32 metadata, quantize through the bucketed path")
    dev = _device()
    codes = torch.from_numpy(np.concatenate([np.asarray(b.codes, dtype=np.int64) for b in blocks])).to(dev)
    meta = torch.tensor([[b.shift, b.scale_lo, b.scale_hi] for b in blocks], dtype=torch.float32, device=dev)
    packed = pack_codes(codes, bit_width, bucket_size)
    msg = encode_segment(packed, meta, total, (bit_width, bucket_size))
    return msg.cpu().numpy().tobytes()


def decode(data: bytes):
    """Exact inverse of encode; malformed input raises a DecodeError (wire.py:134-184)."""
    dev = _device()
    buf = np.frombuffer(bytes(data), dtype=np.uint8)
    msg = torch.from_numpy(buf.copy()).to(dev) if buf.size else torch.empty(0, dtype=torch.uint8, device=dev)
    seg = decode_segment(msg)
    if seg.length == 0:
        return []
    codes = unpack_codes(seg.codes, seg.length, seg.bits, seg.bucket).cpu().numpy().astype(np.uint32)
    meta = seg.meta.cpu().numpy().astype(np.float64)
    blocks = []
    for j in range(meta.shape[0]):
        s = j * seg.bucket
        m = min(seg.bucket, seg.length - s)
        blocks.append(QuantizedBlock(codes[s:s + m], meta[j, 0], meta[j, 1], meta[j, 2], seg.bits, m))
    return blocks
