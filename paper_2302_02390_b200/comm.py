"""One-process-per-GPU quantized collectives (C1 all-gather / C2 reduce-scatter).

:class:`QSDPComm` wraps the C-ABI communicator (include/qsdp_b200.h): every
rank allocates a workspace, exports a CUDA IPC handle, the handles are
exchanged once over ``torch.distributed`` (host plumbing only), and from then
on the data path is the library's own kernels reading peers' HBM over NVLink --
no NCCL call sits on it.

Keys follow the reference protocol (pkg/src/qsdp/sharded.py:323-433):
all-gather buckets are keyed (root, step, layer, phase, worker=0, start) with
the shard's global start; reduce-scatter buckets (root, step, layer,
PHASE_GRAD, worker=rank, start of the destination segment).
"""

from __future__ import annotations

import ctypes

import torch
import torch.distributed as dist

from . import _lib
from .quantize import QuantSpec, SegmentKey, _DTYPE_CODE

__all__ = ["QSDPComm", "plan_segments", "all_gather_plan", "reduce_scatter_plan", "sent_bits"]


def plan_segments(size: int, world: int, pad_to: int = 1):
    """Per-rank (global_start, length) segments of a flat tensor.

    ``pad_to == 1`` reproduces ``shard_bounds`` (sharded.py:193-200: remainder
    to the last rank).  ``pad_to > 1`` gives FSDP2-style equal shards padded to
    a multiple of ``pad_to`` elements (the last ones may be short or empty).
    """
    if world < 1:
        raise ValueError("world must be >= 1")
    if pad_to <= 1:
        base = size // world
        return [(p * base, base if p < world - 1 else size - p * base) for p in range(world)]
    per = -(-size // world)
    per = -(-per // pad_to) * pad_to
    segs = []
    for p in range(world):
        s = min(p * per, size)
        segs.append((s, max(0, min(per, size - s))))
    return segs


def all_gather_plan(rank: int, world: int, segs, key: SegmentKey):
    """What rank ``rank`` does in one quantized all-gather (sharded.py:323-373).

    Returns ``(quantize, pull)``: ``quantize`` = [(global_start, length, key)] for
    its own shard (worker 0, the shard's global start); ``pull`` = [(src_rank,
    out_offset, length)] -- every rank's slot, dequantized into the gathered
    tensor at the segment's offset.  This is the schedule the C ABI executes.
    """
    k = SegmentKey(key.root_seed, key.step, key.layer, key.phase, 0)
    s, n = segs[rank]
    quantize = [(s, n, k)] if n > 0 else []
    base = segs[0][0]
    pull = [(p, segs[p][0] - base, segs[p][1]) for p in range(world) if segs[p][1] > 0]
    return quantize, pull


def reduce_scatter_plan(rank: int, world: int, segs, key: SegmentKey):
    """What rank ``rank`` does in one quantized reduce-scatter (sharded.py:375-433).

    ``quantize`` = [(dst, global_start, length, key)] for every destination
    segment of its gradient (worker = rank); ``pull`` = the sources 0..P-1 whose
    slot ``rank`` are dequant-accumulated in order, then divided by ``world``.
    """
    k = SegmentKey(key.root_seed, key.step, key.layer, key.phase, rank)
    quantize = [(q, segs[q][0], segs[q][1], k) for q in range(world) if segs[q][1] > 0]
    pull = list(range(world)) if segs[rank][1] > 0 else []
    return quantize, pull


def sent_bits(kind: str, rank: int, world: int, segs, spec: QuantSpec) -> int:
    """Wire bits this rank puts on the links for one collective -- the reference
    ledger's records restricted to the sender (sharded.py:349-358, 403-413): an
    all-gather message crosses to world-1 peers, a reduce-scatter segment to its
    owner (the self-contribution is free)."""
    from .quantize import message_size_bits
    if kind == "allgather":
        n = segs[rank][1]
        return message_size_bits(n, spec) * (world - 1) if n > 0 else 0
    return sum(message_size_bits(segs[q][1], spec) for q in range(world) if q != rank and segs[q][1] > 0)


def record_allgather(entry, layer: str, segs, spec: QuantSpec) -> None:
    """The reference's ledger records of one quantized all-gather
    (sharded.py:349-358): one message per non-empty shard, world-1 copies."""
    from .quantize import message_size_bits
    from .sharded import Transfer
    world = len(segs)
    for _, n in segs:
        if n > 0:
            entry.record(Transfer("allgather", layer, spec.bits, message_size_bits(n, spec) // 8, world - 1,
                                  n * spec.bits))
    entry.allgather_events += 1


def record_reducescatter(entry, layer: str, segs, spec: QuantSpec) -> None:
    """The reference's ledger records of one quantized reduce-scatter
    (sharded.py:403-413): every (source p, destination q != p) segment message."""
    from .quantize import message_size_bits
    from .sharded import Transfer
    world = len(segs)
    for q, (_, n) in enumerate(segs):
        if n == 0:
            continue
        for p in range(world):
            if p != q:
                entry.record(Transfer("reducescatter", layer, spec.bits, message_size_bits(n, spec) // 8, 1,
                                      n * spec.bits))
    entry.reducescatter_events += 1


class QSDPComm:
    """NVLink peer-memory communicator for QSDP's quantized AG / RS."""

    def __init__(self, max_segment_elems: int, wspec: QuantSpec, gspec: QuantSpec,
                 group: dist.ProcessGroup | None = None, device: torch.device | None = None,
                 weight_levels=None):
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        if self.world > _lib.MAX_WORLD:
            raise ValueError(f"at most {_lib.MAX_WORLD} ranks per box")
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.wspec, self.gspec = wspec, gspec
        self.max_segment_elems = int(max_segment_elems)
        self._wcfg, self._gcfg = wspec.cfg(), gspec.cfg()
        L = _lib.lib()
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(L.qsdp_comm_create(ctypes.byref(h), self.rank, self.world, self.device.index,
                                          self.max_segment_elems, ctypes.byref(self._wcfg),
                                          ctypes.byref(self._gcfg)))
        self._h = h
        if self.world > 1:
            buf = (ctypes.c_uint8 * _lib.IPC_HANDLE_BYTES)()
            _lib.check(L.qsdp_comm_ipc_handle(self._h, buf))
            mine = bytes(buf)
            allh = [None] * self.world
            dist.all_gather_object(allh, mine, group=group)
            blob = b"".join(allh)
            cb = (ctypes.c_uint8 * len(blob)).from_buffer_copy(blob)
            _lib.check(L.qsdp_comm_open_peers(self._h, cb))
            dist.barrier(group=group)
        if weight_levels is not None:
            self.set_weight_levels(weight_levels)

    def set_weight_levels(self, table) -> None:
        """Learned weight levels: with ``wspec.inner == "levels"``
        the all-gather quantizes / dequantizes through ``table`` (a
        :class:`~.levels.LevelTable` of 2^bits levels, kept on this device)."""
        if self.wspec.inner != "levels":
            raise ValueError("weight spec is not inner='levels'")
        q = table.device(self.device)
        self._wlevels = q  # keep alive while the comm uses it
        _lib.check(_lib.lib().qsdp_comm_set_weight_levels(self._h, q.data_ptr(), q.numel()))

    def set_step_source(self, counter: torch.Tensor | None) -> None:
        """Keys use ``key.step + counter`` read on the device (graph replay)."""
        if counter is not None and (counter.dtype != torch.int64 or counter.device != self.device):
            raise ValueError("step counter must be an int64 tensor on the communicator's device")
        self._step_src = counter  # keep alive
        _lib.check(_lib.lib().qsdp_comm_set_step_source(self._h, counter.data_ptr() if counter is not None else None))

    def set_sm_budget(self, sms: int) -> None:
        """Size this communicator's kernels for at most ``sms`` SMs, so collectives overlapping
        compute on another stream leave it the other SMs (0 = default: the whole GPU at world
        1, all but 8 SMs at world > 1 so other collectives' barriers always find an SM;
        < 0 = the whole GPU)."""
        _lib.check(_lib.lib().qsdp_comm_set_sm_budget(self._h, int(sms)))

    def set_ctas_per_sm(self, ctas: int) -> None:
        """At most ``ctas`` quantizer CTAs per SM (0 = occupancy): an all-gather capped at one
        leaves the other slot of every SM to a concurrent reduce-scatter."""
        _lib.check(_lib.lib().qsdp_comm_set_ctas_per_sm(self._h, int(ctas)))

    def set_timeout(self, ms: int) -> None:
        """Barrier timeout: a peer that does not arrive within ``ms`` milliseconds makes the
        barrier give up instead of hanging; :meth:`check` (and every later collective)
        then raises :class:`~._lib.QSDPError` naming the peer."""
        _lib.check(_lib.lib().qsdp_comm_set_timeout(self._h, int(ms)))

    def check(self) -> None:
        """Raise if a peer missed a barrier of an already-completed collective (does not
        synchronise: call it after the stream has run the collectives)."""
        _lib.check(_lib.lib().qsdp_comm_status(self._h))

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.lib().qsdp_comm_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _segs(self, segs):
        if len(segs) != self.world:
            raise ValueError("need one segment per rank")
        arr = (_lib.Segment * self.world)()
        for p, (s, n) in enumerate(segs):
            arr[p] = _lib.Segment(int(s), int(n))
        return arr

    def all_gather(self, shard: torch.Tensor, segs, key: SegmentKey, out: torch.Tensor) -> torch.Tensor:
        """C1: ``out`` (the full tensor, element 0 = segs[0] start) receives every
        rank's dequantized shard; ``shard`` is this rank's segs[rank] slice."""
        if shard.numel() != segs[self.rank][1]:
            raise ValueError("shard length does not match its segment")
        arr = self._segs(segs)
        k = key.c()
        with torch.cuda.device(self.device):
            _lib.check(_lib.lib().qsdp_all_gather(
                self._h, shard.data_ptr(), _DTYPE_CODE[shard.dtype], arr, ctypes.byref(k), out.data_ptr(),
                _DTYPE_CODE[out.dtype], torch.cuda.current_stream(self.device).cuda_stream))
        return out

    @staticmethod
    def _pieces(pieces):
        arr = (_lib.Piece * len(pieces))()
        for k, pc in enumerate(pieces):
            src, off, n = pc[:3]
            raw = 1 if len(pc) > 3 and pc[3] else 0
            arr[k] = _lib.Piece(src.data_ptr() if src is not None else None, int(off), int(n), raw, 0)
        return arr

    def all_gather_pieces(self, pieces, rank_stride: int, key: SegmentKey, out: torch.Tensor,
                          in_dtype=torch.float32) -> torch.Tensor:
        """C1 over a group of pieces in one call: ``pieces`` = [(this rank's piece tensor, offset,
        numel[, raw])]; rank q's piece k lands at ``out[q * rank_stride + offset]`` (keyed start).
        ``raw`` pieces travel at full precision (cast to ``out.dtype``, sharded.py:359-371)."""
        arr = self._pieces(pieces)
        k = key.c()
        with torch.cuda.device(self.device):
            _lib.check(_lib.lib().qsdp_all_gather_pieces(
                self._h, arr, len(pieces), _DTYPE_CODE[in_dtype], int(rank_stride), ctypes.byref(k), out.data_ptr(),
                _DTYPE_CODE[out.dtype], torch.cuda.current_stream(self.device).cuda_stream))
        return out

    def reduce_scatter_pieces(self, grad: torch.Tensor, pieces, rank_stride: int, key: SegmentKey,
                              out: torch.Tensor) -> torch.Tensor:
        """C2 over a group of pieces: ``grad`` is this rank's rank-major gradient
        [world * rank_stride]; ``pieces`` = [(offset, numel[, raw])]; ``out[offset]`` receives
        piece k's average (``raw``: of the full-precision values, fp64 in rank order,
        sharded.py:414-429)."""
        arr = (_lib.Piece * len(pieces))()
        esz = grad.element_size()
        for j, pc in enumerate(pieces):
            off, n = pc[:2]
            raw = 1 if len(pc) > 2 and pc[2] else 0
            arr[j] = _lib.Piece(grad.data_ptr() + int(off) * esz, int(off), int(n), raw, 0)
        k = key.c()
        with torch.cuda.device(self.device):
            _lib.check(_lib.lib().qsdp_reduce_scatter_pieces(
                self._h, arr, len(pieces), _DTYPE_CODE[grad.dtype], int(rank_stride), ctypes.byref(k), out.data_ptr(),
                _DTYPE_CODE[out.dtype], torch.cuda.current_stream(self.device).cuda_stream))
        return out

    def reduce_scatter_lattice(self, full_grad: torch.Tensor, segs, key: SegmentKey, x_shard: torch.Tensor,
                               step, out: torch.Tensor | None = None) -> torch.Tensor:
        """C2 + the lattice-projected step on this rank's shard, in the K4 epilogue
        (``step`` a :class:`~.lattice.LatticeStep`): ``x_shard``
        moves in place; ``out`` (optional) receives the average gradient."""
        if x_shard.numel() < segs[self.rank][1]:
            raise ValueError("iterate shorter than this rank's segment")
        arr = self._segs(segs)
        k = key.c()
        lat = step.c(x_shard.dtype)
        odt = out.dtype if out is not None else torch.float32
        with torch.cuda.device(self.device):
            _lib.check(_lib.lib().qsdp_reduce_scatter_lattice(
                self._h, full_grad.data_ptr(), _DTYPE_CODE[full_grad.dtype], arr, ctypes.byref(k),
                out.data_ptr() if out is not None else None, _DTYPE_CODE[odt], x_shard.data_ptr(), ctypes.byref(lat),
                torch.cuda.current_stream(self.device).cuda_stream))
        return x_shard

    def reduce_scatter(self, full_grad: torch.Tensor, segs, key: SegmentKey, out: torch.Tensor) -> torch.Tensor:
        """C2: ``out`` (this rank's shard) receives the fp64-ordered average of
        every rank's dequantized contribution to segs[rank]."""
        if out.numel() < segs[self.rank][1]:
            raise ValueError("output shorter than this rank's segment")
        arr = self._segs(segs)
        k = key.c()
        with torch.cuda.device(self.device):
            _lib.check(_lib.lib().qsdp_reduce_scatter(
                self._h, full_grad.data_ptr(), _DTYPE_CODE[full_grad.dtype], arr, ctypes.byref(k),
                out.data_ptr(), _DTYPE_CODE[out.dtype], torch.cuda.current_stream(self.device).cuda_stream))
        return out


def split_segments(segs, bucket: int, chunks: int):
    """Cut every rank's segment into ``chunks`` bucket-aligned sub-segments
    (sub-segment j of each rank covers its buckets [j*nb/chunks, (j+1)*nb/chunks)).
    Keys stay those of the whole collective: a bucket is keyed by its global start,
    so the codes and scales are unchanged (sharded.py:243-248)."""
    out = []
    for j in range(chunks):
        sub = []
        for s, n in segs:
            nb = -(-n // bucket) if n else 0
            b0, b1 = nb * j // chunks, nb * (j + 1) // chunks
            lo, hi = min(n, b0 * bucket), min(n, b1 * bucket)
            sub.append((s + lo, hi - lo))
        out.append(sub)
    return out


class PipelinedComm:
    """C1 / C2 of large tensors as ``chunks`` bucket-aligned sub-collectives that
    alternate between two communicators on two streams, so one chunk's
    quantize + NVLink push overlaps the previous chunk's dequantization (the two
    phases of a single collective cannot overlap each other).  Results are
    bit-identical to one QSDPComm call."""

    def __init__(self, max_segment_elems: int, wspec: QuantSpec, gspec: QuantSpec, chunks: int = 4,
                 group: dist.ProcessGroup | None = None, device: torch.device | None = None):
        self.chunks = max(1, int(chunks))
        sub = -(-int(max_segment_elems) // self.chunks) + max(wspec.bucket, gspec.bucket)
        self.comms = [QSDPComm(sub, wspec, gspec, group=group, device=device) for _ in range(2)]
        self.device = self.comms[0].device
        self.rank = self.comms[0].rank
        self.streams = [torch.cuda.current_stream(self.device), torch.cuda.Stream(device=self.device)]
        self.wspec, self.gspec = wspec, gspec

    def set_step_source(self, counter):
        for c in self.comms:
            c.set_step_source(counter)

    def _run(self, fn):
        main = torch.cuda.current_stream(self.device)
        side = self.streams[1]
        ev = torch.cuda.Event()
        ev.record(main)
        side.wait_event(ev)
        for j in range(self.chunks):
            with torch.cuda.stream(main if j % 2 == 0 else side):
                fn(j, self.comms[j % 2])
        main.wait_stream(side)

    def all_gather(self, shard: torch.Tensor, segs, key: SegmentKey, out: torch.Tensor) -> torch.Tensor:
        parts = split_segments(segs, self.wspec.bucket, self.chunks)
        base = segs[0][0]
        s_me = segs[self.rank][0]

        def one(j, comm):
            sub = parts[j]
            o0 = sub[0][0] - base
            sh = shard[sub[self.rank][0] - s_me: sub[self.rank][0] - s_me + sub[self.rank][1]]
            comm.all_gather(sh, sub, key, out[o0:])
        self._run(one)
        return out

    def reduce_scatter(self, full_grad: torch.Tensor, segs, key: SegmentKey, out: torch.Tensor) -> torch.Tensor:
        parts = split_segments(segs, self.gspec.bucket, self.chunks)
        base = segs[0][0]
        s_me = segs[self.rank][0]

        def one(j, comm):
            sub = parts[j]
            g0 = sub[0][0] - base
            o = out[sub[self.rank][0] - s_me:]
            comm.reduce_scatter(full_grad[g0:], sub, key, o)
        self._run(one)
        return out

    def close(self):
        for c in self.comms:
            c.close()
