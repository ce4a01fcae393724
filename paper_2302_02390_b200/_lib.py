"""ctypes binding of the C ABI in include/qsdp_b200.h (libqsdp_b200.so).

The product path has no fallback: if the shared library is missing or a CUDA
device is absent, calls raise instead of computing anything on the CPU.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
# QSDP_LIB_PATH: an experiment build of the same library (A/B runs); default the in-tree build
LIB_PATH = os.environ.get("QSDP_LIB_PATH") or os.path.join(_HERE, "libqsdp_b200.so")
CSRC = os.path.join(_HERE, "csrc")

QSDP_OK = 0
QSDP_EINVAL = 1
QSDP_ENONFINITE = 2
QSDP_ERANGE = 3
QSDP_ECUDA = 4
QSDP_ENCCL = 5
QSDP_EPEER = 6
QSDP_EDECODE = 7
QSDP_ETRUNC = 8
QSDP_EVERSION = 9

INNER_SHIFT = 0
INNER_STOCHASTIC = 1
INNER_LEVELS = 2
F32, F64, BF16 = 0, 1, 2
IPC_HANDLE_BYTES = 64
MAX_WORLD = 8

EXPORTED_SYMBOLS = (
    "qsdp_num_buckets", "qsdp_codes_bytes", "qsdp_message_size_bits", "qsdp_shard_bounds",
    "qsdp_last_error", "qsdp_version", "qsdp_quantize", "qsdp_quantize_batch", "qsdp_dequantize",
    "qsdp_dequantize_batch", "qsdp_dequant_accumulate", "qsdp_dequant_accumulate_batch",
    "qsdp_wire_encode", "qsdp_comm_create", "qsdp_comm_ipc_handle", "qsdp_comm_open_peers",
    "qsdp_all_gather", "qsdp_reduce_scatter", "qsdp_comm_destroy", "qsdp_quantize_batch_dstep",
    "qsdp_counter_add", "qsdp_comm_set_step_source",
    "qsdp_quantize_levels", "qsdp_quantize_levels_batch", "qsdp_dequantize_levels",
    "qsdp_dequantize_levels_batch", "qsdp_learn_levels", "qsdp_comm_set_weight_levels",
    "qsdp_wire_parse", "qsdp_wire_encode_device", "qsdp_wire_decode_device", "qsdp_pack_codes",
    "qsdp_unpack_codes", "qsdp_dequant_accumulate_lattice", "qsdp_reduce_scatter_lattice",
    "qsdp_comm_set_sm_budget", "qsdp_comm_set_timeout", "qsdp_comm_status", "qsdp_all_gather_pieces",
    "qsdp_reduce_scatter_pieces", "qsdp_quantize_stream", "qsdp_levels_stochastic", "qsdp_comm_set_ctas_per_sm",
)


class Piece(ctypes.Structure):
    _fields_ = [("src", ctypes.c_void_p), ("offset", ctypes.c_int64), ("numel", ctypes.c_int64),
                ("raw", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class QCfg(ctypes.Structure):
    _fields_ = [("bits", ctypes.c_int32), ("bucket", ctypes.c_int32),
                ("inner", ctypes.c_int32), ("noise", ctypes.c_int32)]


class Key(ctypes.Structure):
    _fields_ = [("root_seed", ctypes.c_uint64), ("step", ctypes.c_uint64),
                ("layer", ctypes.c_uint64), ("phase", ctypes.c_uint64),
                ("worker", ctypes.c_uint64)]


class Segment(ctypes.Structure):
    _fields_ = [("global_start", ctypes.c_int64), ("length", ctypes.c_int64)]


class QItem(ctypes.Structure):
    _fields_ = [("x", ctypes.c_void_p), ("seg", Segment), ("key", Key),
                ("codes", ctypes.c_void_p), ("meta", ctypes.c_void_p)]


class DItem(ctypes.Structure):
    _fields_ = [("codes", ctypes.c_void_p * 8), ("meta", ctypes.c_void_p * 8),
                ("nsrc", ctypes.c_int32), ("length", ctypes.c_int64), ("out", ctypes.c_void_p)]


class Lattice(ctypes.Structure):
    _fields_ = [("lr_over_beta", ctypes.c_double), ("delta", ctypes.c_double), ("shift_key", Key),
                ("x_dtype", ctypes.c_int32)]


class WireInfo(ctypes.Structure):
    _fields_ = [("version", ctypes.c_int32), ("bits", ctypes.c_int32), ("bucket", ctypes.c_int64),
                ("blocks", ctypes.c_int64), ("total_length", ctypes.c_int64), ("expected_bytes", ctypes.c_int64),
                ("complete_blocks", ctypes.c_int64)]


class QSDPError(RuntimeError):
    """CUDA / peer failure inside the native library."""


# The reference's wire exception hierarchy (wire.py:54-75).
class WireError(ValueError):
    pass


class EncodeError(WireError):
    pass


class DecodeError(WireError):
    pass


class TruncatedMessageError(DecodeError):
    pass


class UnsupportedVersionError(DecodeError):
    pass


class CodeRangeError(DecodeError):
    pass


_lib = None


def build(jobs: int = 4) -> str:
    """Compile libqsdp_b200.so for sm_100a (nvcc; no GPU needed)."""
    subprocess.run(["make", "-s", f"-j{jobs}", "-C", CSRC], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make -C {CSRC}` (or __graft_entry__.build()). "
            "There is no CPU fallback for the QSDP hot path.")
    L = ctypes.CDLL(LIB_PATH)
    i64, i32, vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
    cfgp = ctypes.POINTER(QCfg)
    keyp = ctypes.POINTER(Key)
    segp = ctypes.POINTER(Segment)
    L.qsdp_num_buckets.argtypes = [i64, i32]
    L.qsdp_num_buckets.restype = i64
    L.qsdp_codes_bytes.argtypes = [i64, cfgp]
    L.qsdp_codes_bytes.restype = i64
    L.qsdp_message_size_bits.argtypes = [i64, cfgp]
    L.qsdp_message_size_bits.restype = i64
    L.qsdp_shard_bounds.argtypes = [i64, i32, segp]
    L.qsdp_shard_bounds.restype = None
    L.qsdp_last_error.restype = ctypes.c_char_p
    L.qsdp_version.restype = ctypes.c_char_p
    L.qsdp_quantize.argtypes = [vp, i32, Segment, cfgp, keyp, vp, vp, vp, vp]
    L.qsdp_quantize_batch.argtypes = [ctypes.POINTER(QItem), i32, i32, cfgp, vp, vp]
    L.qsdp_quantize_batch_dstep.argtypes = [ctypes.POINTER(QItem), i32, i32, cfgp, vp, vp, vp]
    L.qsdp_counter_add.argtypes = [vp, ctypes.c_uint64, vp]
    L.qsdp_comm_set_step_source.argtypes = [vp, vp]
    L.qsdp_comm_set_weight_levels.argtypes = [vp, vp, i32]
    L.qsdp_comm_set_sm_budget.argtypes = [vp, i32]
    L.qsdp_comm_set_ctas_per_sm.argtypes = [vp, i32]
    L.qsdp_comm_set_timeout.argtypes = [vp, i64]
    L.qsdp_comm_status.argtypes = [vp]
    L.qsdp_quantize_stream.argtypes = [vp, i32, i64, cfgp, vp, vp, vp, vp, vp]
    L.qsdp_levels_stochastic.argtypes = [vp, i64, vp, i32, vp, vp, vp]
    L.qsdp_all_gather_pieces.argtypes = [vp, ctypes.POINTER(Piece), i32, i32, i64, keyp, vp, i32, vp]
    L.qsdp_reduce_scatter_pieces.argtypes = [vp, ctypes.POINTER(Piece), i32, i32, i64, keyp, vp, i32, vp]
    L.qsdp_wire_parse.argtypes = [vp, i64, ctypes.POINTER(WireInfo)]
    L.qsdp_wire_encode_device.argtypes = [vp, vp, i64, cfgp, vp, i64, vp]
    L.qsdp_wire_decode_device.argtypes = [vp, ctypes.POINTER(WireInfo), vp, vp, vp, vp]
    L.qsdp_pack_codes.argtypes = [vp, i64, cfgp, vp, vp]
    L.qsdp_dequant_accumulate_lattice.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(vp), i32, i64, cfgp, i32, vp,
                                                  i32, vp, ctypes.POINTER(Lattice), vp]
    L.qsdp_reduce_scatter_lattice.argtypes = [vp, vp, i32, segp, keyp, vp, i32, vp, ctypes.POINTER(Lattice), vp]
    L.qsdp_unpack_codes.argtypes = [vp, i64, cfgp, vp, vp]
    L.qsdp_dequantize.argtypes = [vp, vp, i64, cfgp, vp, i32, vp]
    L.qsdp_dequantize_batch.argtypes = [ctypes.POINTER(DItem), i32, cfgp, i32, vp]
    L.qsdp_dequant_accumulate.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(vp), i32, i64, cfgp,
                                          i32, vp, i32, vp]
    L.qsdp_dequant_accumulate_batch.argtypes = [ctypes.POINTER(DItem), i32, cfgp, i32, i32, vp]
    L.qsdp_wire_encode.argtypes = [vp, vp, i64, cfgp, vp, i64]
    L.qsdp_wire_encode.restype = i64
    L.qsdp_comm_create.argtypes = [ctypes.POINTER(vp), i32, i32, i32, i64, cfgp, cfgp]
    L.qsdp_comm_ipc_handle.argtypes = [vp, vp]
    L.qsdp_comm_open_peers.argtypes = [vp, vp]
    L.qsdp_all_gather.argtypes = [vp, vp, i32, segp, keyp, vp, i32, vp]
    L.qsdp_reduce_scatter.argtypes = [vp, vp, i32, segp, keyp, vp, i32, vp]
    L.qsdp_comm_destroy.argtypes = [vp]
    L.qsdp_quantize_levels.argtypes = [vp, i32, i64, cfgp, vp, i32, vp, vp, vp, vp]
    L.qsdp_quantize_levels_batch.argtypes = [ctypes.POINTER(QItem), i32, i32, cfgp, vp, i32, vp, vp]
    L.qsdp_dequantize_levels.argtypes = [vp, vp, i64, cfgp, vp, i32, vp, i32, vp]
    L.qsdp_dequantize_levels_batch.argtypes = [ctypes.POINTER(DItem), i32, cfgp, vp, i32, i32, vp]
    L.qsdp_learn_levels.argtypes = [vp, i64, vp, i32, ctypes.c_double, vp]
    for name in ("qsdp_quantize", "qsdp_quantize_batch", "qsdp_quantize_batch_dstep", "qsdp_counter_add",
                 "qsdp_comm_set_step_source", "qsdp_dequantize", "qsdp_dequantize_batch",
                 "qsdp_dequant_accumulate", "qsdp_dequant_accumulate_batch", "qsdp_comm_create",
                 "qsdp_comm_ipc_handle", "qsdp_comm_open_peers", "qsdp_all_gather",
                 "qsdp_reduce_scatter", "qsdp_comm_destroy", "qsdp_quantize_levels",
                 "qsdp_quantize_levels_batch", "qsdp_dequantize_levels", "qsdp_dequantize_levels_batch",
                 "qsdp_learn_levels", "qsdp_comm_set_weight_levels", "qsdp_wire_parse",
                 "qsdp_wire_encode_device", "qsdp_wire_decode_device", "qsdp_pack_codes", "qsdp_unpack_codes",
                 "qsdp_dequant_accumulate_lattice", "qsdp_reduce_scatter_lattice", "qsdp_comm_set_sm_budget",
                 "qsdp_comm_set_timeout", "qsdp_comm_status", "qsdp_all_gather_pieces", "qsdp_reduce_scatter_pieces",
                 "qsdp_quantize_stream", "qsdp_levels_stochastic", "qsdp_comm_set_ctas_per_sm"):
        getattr(L, name).restype = ctypes.c_int
    _lib = L
    return _lib


_hot = None


def hot():
    """The group collectives through a ``ctypes.PyDLL`` view of the same library: the call
    keeps the GIL.  They only enqueue launches (~15-20 us, never block), and FSDP2 drives them
    from its hooks on the main and autograd threads; a GIL release per call let the other
    thread take the interpreter for up to the switch interval before the hook could resume
    (measured 109 vs 17 us per all-gather call inside the 1.3B step)."""
    global _hot
    if _hot is None:
        lib()  # existence check, error message
        H = ctypes.PyDLL(LIB_PATH)
        vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        for name in ("qsdp_all_gather_pieces", "qsdp_reduce_scatter_pieces"):
            f = getattr(H, name)
            f.argtypes = [vp, ctypes.POINTER(Piece), i32, i32, i64, ctypes.POINTER(Key), vp, i32, vp]
            f.restype = ctypes.c_int
        _hot = H
    return _hot


def check(status: int) -> None:
    """Map a qsdp_status to the reference's exception types."""
    if status == QSDP_OK:
        return
    msg = lib().qsdp_last_error().decode(errors="replace")
    if status in (QSDP_EINVAL, QSDP_ENONFINITE):
        raise ValueError(msg)
    if status == QSDP_ERANGE:
        raise CodeRangeError(msg)
    if status == QSDP_EDECODE:
        raise DecodeError(msg)
    if status == QSDP_ETRUNC:
        raise TruncatedMessageError(msg)
    if status == QSDP_EVERSION:
        raise UnsupportedVersionError(msg)
    raise QSDPError(f"qsdp status {status}: {msg}")
