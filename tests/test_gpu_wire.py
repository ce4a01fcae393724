"""GPU wire codec vs the reference's messages (tests/golden) and
its decode behaviour; restates the reference's test_wire.py cases."""

import numpy as np
import pytest
import torch

from conftest import golden_cases

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def W():
    from paper_2302_02390_b200 import wire
    return wire


def _blocks(oracle, c):
    from paper_2302_02390_b200.quantize import QuantizedBlock
    out, S = [], c["bucket"]
    pbs = (S * c["bits"] + 7) // 8
    for j, m in enumerate(c["meta"].astype(np.float64)):
        n = min(S, c["n"] - j * S)
        cj = oracle.unpack(c["codes"][j * pbs: j * pbs + (n * c["bits"] + 7) // 8], n, c["bits"])
        out.append(QuantizedBlock(cj, m[0], m[1], m[2], c["bits"], n))
    return out


def test_device_codec_matches_golden_messages(golden, W):
    from paper_2302_02390_b200.quantize import QuantSpec
    n = 0
    for c in golden_cases(golden):
        spec = QuantSpec(c["bits"], c["bucket"], "shift")
        codes = torch.from_numpy(c["codes"].copy()).cuda()
        meta = torch.from_numpy(c["meta"].copy()).cuda()
        msg = W.encode_segment(codes, meta, c["n"], spec)
        assert msg.cpu().numpy().tobytes() == c["wire"].tobytes(), f"case {c['i']}"
        seg = W.decode_segment(torch.from_numpy(c["wire"].copy()).cuda())
        assert (seg.length, seg.bits) == (c["n"], c["bits"])
        assert np.array_equal(seg.codes.cpu().numpy(), c["codes"])
        assert np.array_equal(seg.meta.cpu().numpy(), c["meta"])
        n += 1
    assert n >= 50


def test_reference_api_matches_golden(golden, oracle, W):
    for c in list(golden_cases(golden))[::3]:
        blocks = _blocks(oracle, c)
        assert W.encode(blocks) == c["wire"].tobytes()
        assert W.decode(c["wire"].tobytes()) == blocks
        assert W.message_size_bits(blocks) == len(c["wire"]) * 8


def test_decode_errors_match_reference(golden, W):
    """Malformed messages raise what the reference decode raises (class by class)."""
    for i in range(int(golden["wire_n"])):
        msg = bytes(golden[f"wire_{i}_msg"].tobytes())
        want = str(golden[f"wire_{i}_res"])
        try:
            W.decode(msg)
            got = "ok"
        except Exception as e:  # noqa: BLE001
            got = type(e).__name__
        assert got == want, f"wire case {i}: {got} != {want}"


def _block(codes, bits, shift=0.0, lo=0.0, hi=1.0):
    from paper_2302_02390_b200.quantize import QuantizedBlock
    c = np.asarray(codes, dtype=np.uint32)
    return QuantizedBlock(c, shift, lo, hi, bits, c.size)


def _random_block_list(rng, max_bits=16):
    from paper_2302_02390_b200.quantize import QuantizedBlock
    bits = int(rng.integers(1, max_bits + 1))
    bucket = int(rng.integers(1, 40))
    count = int(rng.integers(1, 5))
    last = int(rng.integers(1, bucket + 1))
    out = []
    for i in range(count):
        n = bucket if i < count - 1 else last
        out.append(QuantizedBlock(rng.integers(0, 1 << bits, n, dtype=np.uint64).astype(np.uint32),
                                  float(np.float32(rng.normal())), float(np.float32(-abs(rng.normal()))),
                                  float(np.float32(abs(rng.normal()) + 1)), bits, n))
    return out


def test_fuzzed_round_trips(W):
    """reference test_wire.py:83-97 (fewer iterations: each is a device round trip)."""
    rng = np.random.default_rng(7)
    for _ in range(200):
        blocks = _random_block_list(rng)
        data = W.encode(blocks)
        assert W.message_size_bits(blocks) == len(data) * 8
        assert W.decode(data) == blocks
    for _ in range(30):  # widths 17..32 (QuantizedBlock allows them; the quantizers never emit them)
        blocks = _random_block_list(rng, 32)
        assert W.decode(W.encode(blocks)) == blocks


def test_reference_kats(W):
    from paper_2302_02390_b200.wire import (BLOCK_META_BITS, HEADER_BITS, CodeRangeError, DecodeError, EncodeError,
                                            TruncatedMessageError, UnsupportedVersionError)
    assert len(W.encode([_block(np.arange(8), 4)])) - (HEADER_BITS + BLOCK_META_BITS) // 8 == 4
    assert len(W.encode([_block([1, 2, 3], 3)])) - (HEADER_BITS + BLOCK_META_BITS) // 8 == 2
    assert len(W.encode([])) * 8 == HEADER_BITS and W.decode(W.encode([])) == []
    blocks = [_block([1, 2, 3, 4, 5], 3)]
    data = bytearray(W.encode(blocks))
    start = (HEADER_BITS + BLOCK_META_BITS) // 8
    for bit in range(15):  # every code bit flip changes a code
        d = bytearray(data)
        d[start + bit // 8] ^= 1 << (bit % 8)
        assert W.decode(bytes(d)) != blocks
    d = bytearray(data)
    d[-1] ^= 0x80
    with pytest.raises(DecodeError):
        W.decode(bytes(d))
    d = bytearray(W.encode([_block([1], 2)]))
    d[0] = 9
    with pytest.raises(UnsupportedVersionError):
        W.decode(bytes(d))
    with pytest.raises(TruncatedMessageError):
        W.decode(b"\x01\x02")
    with pytest.raises(TruncatedMessageError):
        W.decode(W.encode([_block(np.arange(8), 4)])[:-1])
    with pytest.raises(DecodeError):
        W.decode(W.encode([_block(np.arange(8), 4)]) + b"\x00")
    d = bytearray(W.encode([_block([1], 2)]))
    d[1] = 40
    with pytest.raises(CodeRangeError):
        W.decode(bytes(d))
    with pytest.raises(EncodeError):
        W.encode([_block([1], 2), _block([1], 3)])
    with pytest.raises(EncodeError):
        W.encode([_block([1, 2], 4), _block([1, 2, 3], 4)])
    with pytest.raises(EncodeError):
        W.encode([_block([1], 4, lo=0.1000000000000001, hi=1.0)])


def test_full_size_round_trip(oracle, W):
    """GPT-2 wte-sized segment: quantize -> encode -> decode -> identical device
    layout, message bytes equal to the oracle's encoder on a prefix bucket set."""
    from paper_2302_02390_b200.quantize import QuantSpec, SegmentKey, quantize_segment
    n = 38633472 + 17
    spec = QuantSpec(8, 1024, "shift")
    x = torch.randn(n, device="cuda") * 0.02
    codes, meta = quantize_segment(x, 0, spec, SegmentKey(0, 3, 0, 0, 0))
    msg = W.encode_segment(codes, meta, n, spec)
    seg = W.decode_segment(msg)
    assert torch.equal(seg.codes, codes) and torch.equal(seg.meta, meta) and seg.length == n
    # the first 5 blocks of the message == the oracle's encoder on those buckets (headers differ)
    cpu = oracle.encode_segment(codes[:5 * 1024].cpu().numpy(), meta[:5].cpu().numpy(), 5 * 1024, 1024, 8)
    assert msg[14:len(cpu)].cpu().numpy().tobytes() == cpu[14:]
