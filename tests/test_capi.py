"""CPU: the C-ABI library loads, exports every symbol include/qsdp_b200.h
declares, and its host-only functions (sizes, ledger accounting, shard bounds,
wire export) agree with the oracle and the reference's known answers."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden_cases
from paper_2302_02390_b200 import _lib

HEADER = os.path.join(ROOT, "include", "qsdp_b200.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(qsdp_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_what_binding_expects():
    assert set(_declared()) == set(_lib.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    for name in _declared():
        assert hasattr(L, name), name
    assert b"sm_100a" in L.qsdp_version()


def _cfg(bits, bucket, inner=0):
    return _lib.QCfg(bits, bucket, inner, 0)


def test_sizes_match_reference_kats(oracle):
    L = _lib.lib()
    # pkg/tests/test_wire.py:50-69 and test_sharded.py:173-183 (dense0: 14+12+1024 B)
    assert L.qsdp_codes_bytes(8, ctypes.byref(_cfg(4, 8))) == 4
    assert L.qsdp_codes_bytes(3, ctypes.byref(_cfg(3, 3))) == 2
    assert L.qsdp_message_size_bits(1024, ctypes.byref(_cfg(8, 1024))) == 8192 + 96 + 112
    assert L.qsdp_message_size_bits(0, ctypes.byref(_cfg(8, 1024))) == 112
    assert L.qsdp_message_size_bits(1024, ctypes.byref(_cfg(8, 1024))) // 8 == 14 + 12 + 1024
    rng = np.random.default_rng(0)
    for _ in range(200):
        n, S, b = int(rng.integers(0, 10**6)), int(rng.integers(1, 5000)), int(rng.integers(1, 17))
        assert L.qsdp_num_buckets(n, S) == (oracle.num_buckets(n, S) if n else 0)
        assert L.qsdp_codes_bytes(n, ctypes.byref(_cfg(b, S))) == (oracle.codes_bytes(n, S, b) if n else 0)
        assert L.qsdp_message_size_bits(n, ctypes.byref(_cfg(b, S))) == oracle.message_size_bits(n, S, b)


def test_shard_bounds_match_reference():
    L = _lib.lib()
    for size, P in [(100, 4), (10, 4), (7, 1), (3, 8), (4096, 3)]:
        arr = (_lib.Segment * P)()
        L.qsdp_shard_bounds(size, P, arr)
        base = size // P
        exp = [(p * base, (p + 1) * base) for p in range(P - 1)] + [((P - 1) * base, size)]
        assert [(a.global_start, a.global_start + a.length) for a in arr] == exp


def test_wire_export_matches_reference_bytes(golden):
    L = _lib.lib()
    for c in golden_cases(golden):
        cfg = _cfg(c["bits"], c["bucket"], c["inner"])
        out = np.zeros(c["wire"].size + 8, dtype=np.uint8)
        codes = np.ascontiguousarray(c["codes"])
        meta = np.ascontiguousarray(c["meta"], dtype=np.float32)
        n = L.qsdp_wire_encode(codes.ctypes.data, meta.ctypes.data, c["n"], ctypes.byref(cfg),
                               out.ctypes.data, out.size)
        assert out[:n].tobytes() == c["wire"].tobytes()


def test_invalid_config_is_value_error_without_gpu():
    L = _lib.lib()
    bad = _cfg(17, 1024)
    st = L.qsdp_quantize(None, 0, _lib.Segment(0, 0), ctypes.byref(bad), ctypes.byref(_lib.Key()),
                         None, None, None, None)
    assert st == _lib.QSDP_EINVAL
    with pytest.raises(ValueError, match="bit_width"):
        _lib.check(st)


def test_ledger_csv_matches_reference_bytes(golden, tmp_path):
    """CommLedger.to_csv is byte-identical to the reference's (sharded.py:161-181)."""
    from paper_2302_02390_b200.sharded import CommLedger, LedgerEntry
    bits = golden["run_0_bits"]
    led = CommLedger()
    for t in range(bits.shape[1]):
        led.append(LedgerEntry(step=t, allgather_bits=int(bits[0, t]), reducescatter_bits=int(bits[1, t])))
    path = tmp_path / "ledger.csv"
    led.to_csv(path)
    assert path.read_bytes() == bytes(golden["ledger_csv"])


def test_collective_ledger_records(oracle):
    """record_allgather / record_reducescatter charge the reference's message sizes
    (sharded.py:349-358, 403-413) for any segmentation."""
    from paper_2302_02390_b200.comm import record_allgather, record_reducescatter
    from paper_2302_02390_b200.quantize import QuantSpec
    from paper_2302_02390_b200.sharded import LedgerEntry
    rng = np.random.default_rng(4)
    for _ in range(20):
        P = int(rng.integers(1, 9))
        segs = [(0, int(n)) for n in rng.integers(0, 5000, P)]
        spec = QuantSpec(int(rng.integers(1, 17)), int(rng.integers(1, 2000)), "shift")
        e = LedgerEntry(step=0)
        record_allgather(e, "w", segs, spec)
        record_reducescatter(e, "w", segs, spec)
        msg = [oracle.message_size_bits(n, spec.bucket, spec.bits) if n else 0 for _, n in segs]
        assert e.allgather_bits == sum(m * (P - 1) for m in msg)
        assert e.reducescatter_bits == sum(m * (P - 1) for m in msg)
        assert e.allgather_payload_bits == sum(n * spec.bits * (P - 1) for _, n in segs)
        assert e.allgather_events == e.reducescatter_events == 1
