"""QSDP protocol hooks on B200: the reference's FSDP-hook API, GPU-backed.

Mirrors pkg/src/qsdp/sharded.py of the reference:

* constants ``PHASE_W_FWD/PHASE_W_BWD/PHASE_GRAD`` (sharded.py:56-58),
  ``QuantConfig`` (:76-93), ``shard_bounds`` (:193-200), ``Transfer`` /
  ``LedgerEntry`` (:115-158) with identical accounting and ``CommLedger``
  (:161-181) with a byte-identical CSV export;
* :class:`QSDPHooks` -- ``_gather(step, layer_idx, phase, entry)`` and
  ``_reduce_scatter(step, layer_idx, per_worker_grads, entry)`` with the exact
  signatures, semantics, keys and ledger records of ``ShardedMLP._gather``
  (:323-373) and ``ShardedMLP._reduce_scatter`` (:375-433).  Mix it into any
  object exposing the ShardedMLP attributes (``layers``, ``cfg.P``,
  ``cfg.root_seed``, ``quant``, ``model.bounds``, ``model.shards``) -- including
  the reference class itself -- and the simulated collectives
  run on the GPU: all P virtual ranks' segments are quantized in one batched
  launch (K1/K2), then dequantized (K3) / dequant-accumulated in source order
  (K4).  Real one-process-per-GPU collectives are in :mod:`.comm`.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .quantize import QuantSpec, SegmentKey, dequant_accumulate, dequantize_segments, \
    message_size_bits, quantize_segments

__all__ = ["PHASE_W_FWD", "PHASE_W_BWD", "PHASE_GRAD", "QuantConfig", "LayerSpec", "Transfer",
           "LedgerEntry", "CommLedger", "shard_bounds", "QSDPHooks", "gather_segments", "reduce_scatter_segments"]

PHASE_W_FWD = 0
PHASE_W_BWD = 1
PHASE_GRAD = 2


@dataclass(frozen=True)
class LayerSpec:
    name: str
    kind: str  # dense | bias | norm
    shape: tuple

    def __post_init__(self):
        if self.kind not in ("dense", "bias", "norm"):
            raise ValueError(f"unknown layer kind {self.kind!r}")

    @property
    def size(self) -> int:
        return int(np.prod(self.shape))


@dataclass(frozen=True)
class QuantConfig:
    """Same fields and validation as the reference QuantConfig (sharded.py:76-93)."""

    quantize_weights: bool = True
    quantize_gradients: bool = True
    weight_bits: int = 8
    gradient_bits: int = 8
    bucket_size: int = 1024
    raw_bits: int = 32
    raw_gradient_bits: int = 32

    def __post_init__(self):
        for name in ("weight_bits", "gradient_bits"):
            if not 1 <= getattr(self, name) <= 16:
                raise ValueError(f"{name} must be in [1, 16]")
        if self.bucket_size < 1:
            raise ValueError("bucket_size must be >= 1")
        if self.raw_bits % 8 or self.raw_gradient_bits % 8:
            raise ValueError("raw transfer widths must be whole bytes")

    def weight_spec(self) -> QuantSpec:
        return QuantSpec(self.weight_bits, self.bucket_size, "shift")

    def gradient_spec(self) -> QuantSpec:
        return QuantSpec(self.gradient_bits, self.bucket_size, "uniform_stochastic")


@dataclass
class Transfer:
    collective: str
    layer: str
    bit_width: int
    nbytes: int
    copies: int
    payload_bits: int

    @property
    def total_bits(self) -> int:
        return self.nbytes * 8 * self.copies


@dataclass
class LedgerEntry:
    step: int
    allgather_bits: int = 0
    reducescatter_bits: int = 0
    allgather_payload_bits: int = 0
    reducescatter_payload_bits: int = 0
    allgather_events: int = 0
    reducescatter_events: int = 0
    transfers: list = field(default_factory=list)
    step_time_s: float = 0.0

    @property
    def total_bits(self) -> int:
        return self.allgather_bits + self.reducescatter_bits

    @property
    def collective_count(self) -> int:
        return self.allgather_events + self.reducescatter_events

    def record(self, t: Transfer) -> None:
        self.transfers.append(t)
        if t.collective == "allgather":
            self.allgather_bits += t.total_bits
            self.allgather_payload_bits += t.payload_bits * t.copies
        else:
            self.reducescatter_bits += t.total_bits
            self.reducescatter_payload_bits += t.payload_bits * t.copies


class CommLedger:
    """Per-step communication record with CSV export (sharded.py:161-181)."""

    def __init__(self):
        self.entries: list = []

    def append(self, entry: LedgerEntry) -> None:
        self.entries.append(entry)

    def to_csv(self, path, no_timestamp: bool = True) -> None:
        import csv
        with open(path, "w", newline="") as fh:
            if not no_timestamp:
                import datetime
                fh.write(f"# generated {datetime.datetime.now().isoformat()}\n")
            w = csv.writer(fh)
            w.writerow(["step", "allgather_bits", "reducescatter_bits", "step_time_s"])
            for e in self.entries:
                w.writerow([e.step, e.allgather_bits, e.reducescatter_bits, repr(e.step_time_s)])


def shard_bounds(size: int, P: int):
    """Contiguous partition, remainder to the last worker (sharded.py:193-200)."""
    if P < 1:
        raise ValueError("P must be >= 1")
    base = size // P
    out = [(p * base, (p + 1) * base) for p in range(P - 1)]
    out.append(((P - 1) * base, size))
    return out


def gather_segments(full_src: torch.Tensor, bounds, spec: QuantSpec, key: SegmentKey,
                    out_dtype=None) -> torch.Tensor:
    """Quantized all-gather of one flat tensor over P virtual ranks on one GPU.

    ``full_src`` holds the concatenated shards (rank p's shard at bounds[p]);
    every shard is quantized with worker 0 keys and its own global start, then
    dequantized into the gathered output (sharded.py:329-358).
    """
    out = torch.empty(full_src.numel(), dtype=out_dtype or full_src.dtype, device=full_src.device)
    items = [(full_src[s:e], s, key) for s, e in bounds if e > s]
    q = quantize_segments(items, spec, check_finite=True)
    jobs = [(c, m, e - s, out[s:e]) for (c, m), (s, e) in zip(q, [b for b in bounds if b[1] > b[0]])]
    dequantize_segments(jobs, spec, out.dtype)
    return out


def reduce_scatter_segments(grads: torch.Tensor, bounds, spec: QuantSpec, root_seed: int, step: int,
                            layer_idx: int, out_dtype=None):
    """Quantized reduce-scatter over P virtual ranks: ``grads`` is [P, size]
    (rank p's full gradient in row p).  Destination q receives
    ``(0 + sum_p dequant(Q(grads[p][s_q:e_q]; worker p))) / P`` (sharded.py:381-431)."""
    P = grads.shape[0]
    items, where = [], []
    for q, (s, e) in enumerate(bounds):
        if e == s:
            continue
        for p in range(P):
            items.append((grads[p, s:e], s, SegmentKey(root_seed, step, layer_idx, PHASE_GRAD, p)))
            where.append((q, p))
    qres = quantize_segments(items, spec, check_finite=True)
    by_q = {}
    for (q, p), cm in zip(where, qres):
        by_q.setdefault(q, []).append(cm)
    outs = []
    dt = out_dtype or grads.dtype
    for q, (s, e) in enumerate(bounds):
        if e == s:
            outs.append(torch.zeros(0, dtype=dt, device=grads.device))
            continue
        outs.append(dequant_accumulate(by_q[q], e - s, spec, P, dtype=dt))
    return outs


class QSDPHooks:
    """Drop-in ``_gather`` / ``_reduce_scatter`` for a ShardedMLP-shaped object.

    Shards live wherever the host keeps them (the reference keeps float64
    numpy arrays); each hook call stages them to the current CUDA device, runs
    the quantized collective there, and returns float64 numpy arrays, bit-equal
    to the reference's (tests/test_gpu_protocol.py).
    """

    qsdp_device: torch.device | None = None

    def _qsdp_dev(self) -> torch.device:
        if self.qsdp_device is None:
            if not torch.cuda.is_available():
                raise RuntimeError("QSDPHooks need a CUDA device (no CPU fallback)")
            self.qsdp_device = torch.device("cuda", torch.cuda.current_device())
        return self.qsdp_device

    def _qsdp_quant(self) -> QuantConfig:
        return self.quant

    def _gather(self, step: int, layer_idx: int, phase: int, entry) -> np.ndarray:
        layer = self.layers[layer_idx]
        P = self.cfg.P
        quant = self._qsdp_quant()
        quantized = layer.kind == "dense" and quant.quantize_weights
        bounds = self.model.bounds[layer.name]
        shards = self.model.shards[layer.name]
        dev = self._qsdp_dev()
        full = torch.from_numpy(np.ascontiguousarray(np.concatenate(shards), dtype=np.float64)).to(dev)
        if quantized:
            spec = QuantSpec(quant.weight_bits, quant.bucket_size, "shift")
            out = gather_segments(full, bounds, spec,
                                  SegmentKey(self.cfg.root_seed, step, layer_idx, phase, 0))
            for s, e in bounds:
                if e > s:
                    entry.record(Transfer("allgather", layer.name, quant.weight_bits,
                                          message_size_bits(e - s, spec) // 8, P - 1,
                                          (e - s) * quant.weight_bits))
        else:
            out = full.clone()  # full-precision path (sharded.py:359-371)
            width = quant.raw_bits if layer.kind == "dense" else 32
            for s, e in bounds:
                if e > s:
                    entry.record(Transfer("allgather", layer.name, width, (e - s) * width // 8, P - 1,
                                          (e - s) * width))
        entry.allgather_events += 1
        return out.cpu().numpy()

    def _reduce_scatter(self, step: int, layer_idx: int, per_worker_grads, entry):
        layer = self.layers[layer_idx]
        P = self.cfg.P
        quant = self._qsdp_quant()
        quantized = layer.kind == "dense" and quant.quantize_gradients
        bounds = self.model.bounds[layer.name]
        dev = self._qsdp_dev()
        g = torch.from_numpy(np.ascontiguousarray(np.stack([np.asarray(x, dtype=np.float64).ravel()
                                                            for x in per_worker_grads]))).to(dev)
        if quantized:
            spec = QuantSpec(quant.gradient_bits, quant.bucket_size, "uniform_stochastic")
            outs = reduce_scatter_segments(g, bounds, spec, self.cfg.root_seed, step, layer_idx)
            for q, (s, e) in enumerate(bounds):
                if e == s:
                    continue
                for p in range(P):
                    if p != q:
                        entry.record(Transfer("reducescatter", layer.name, quant.gradient_bits,
                                              message_size_bits(e - s, spec) // 8, 1,
                                              (e - s) * quant.gradient_bits))
        else:
            width = quant.raw_gradient_bits if layer.kind == "dense" else 32
            outs = []
            for q, (s, e) in enumerate(bounds):
                if e == s:
                    outs.append(torch.zeros(0, dtype=torch.float64, device=dev))
                    continue
                acc = torch.zeros(e - s, dtype=torch.float64, device=dev)
                for p in range(P):
                    acc = acc + g[p, s:e]  # ordered fp64 sum, then /P (sharded.py:430-431)
                    if p != q:
                        entry.record(Transfer("reducescatter", layer.name, width, (e - s) * width // 8, 1,
                                              (e - s) * width))
                # tensor/tensor true division (torch turns `/ python_scalar` into a
                # reciprocal multiply on CUDA, which is not the reference's acc / P)
                outs.append(torch.div(acc, torch.full_like(acc, float(P))))
        entry.reducescatter_events += 1
        return [o.cpu().numpy() for o in outs]
