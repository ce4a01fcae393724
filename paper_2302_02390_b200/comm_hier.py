"""Hierarchical multi-node C1 / C2: quantize once, exchange
codes in two levels -- across nodes (InfiniBand in a cluster) and inside each
node (NVLink) -- and dequantize with the same K1-K4 kernels.

The reference protocol (pkg/src/qsdp/sharded.py:323-433) is topology-free: rank
p's shard is quantized once with key worker 0 (all-gather) and every gradient
segment once with key worker p (reduce-scatter); owners sum the P dequantized
contributions in source order.  Only codes + scales ever travel, so the result
is bit-identical to the single-box communicator and to the oracle whatever the
topology (tests/dist_hier_check.py).

Ranks are grouped into nodes of ``node_size`` consecutive ranks.

* C1: quantize own shard (K1) into a fixed-size slot of packed codes + meta;
  (1) all-gather the slots across nodes among ranks with the same local index
  (one message per node crosses the inter-node fabric per rank); (2) all-gather
  the node-gathered slots inside the node; dequantize all P shards (K3, one
  batched launch).
* C2: quantize the P destination segments (K2) into P slots; (1) inside the
  node, all-to-all so that the local rank with local index ``l`` holds every
  slot destined to the ranks of local index ``l`` in all nodes; (2) across nodes,
  all-to-all among equal local indices delivers each slot to its owner; the
  owner dequant-accumulates the P sources in rank order (K4).

The byte exchanges use NCCL through torch.distributed (NVLink / NVSwitch inside
a node, the inter-node fabric across), on the caller's stream.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from .quantize import (QuantSpec, SegmentKey, codes_bytes, dequant_accumulate, dequantize_segments, num_buckets,
                       quantize_segments)

__all__ = ["HierComm"]


def _slot_bytes(max_seg: int, spec: QuantSpec) -> int:
    c = codes_bytes(max_seg, spec)
    m = 12 * num_buckets(max_seg, spec.bucket)
    return (c + 255) // 256 * 256 + (m + 255) // 256 * 256


class HierComm:
    """Two-level quantized all-gather / reduce-scatter for multi-node jobs."""

    def __init__(self, max_segment_elems: int, wspec: QuantSpec, gspec: QuantSpec, node_size: int,
                 device: torch.device | None = None):
        if not dist.is_initialized():
            raise RuntimeError("HierComm needs torch.distributed (one process per GPU)")
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        if node_size < 1 or self.world % node_size:
            raise ValueError("world size must be a multiple of node_size")
        self.node_size = node_size
        self.nodes = self.world // node_size
        self.node, self.local = divmod(self.rank, node_size)
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.wspec, self.gspec = wspec, gspec
        self.max_seg = int(max_segment_elems)
        # every rank creates every group in the same order (torch.distributed contract)
        self.node_group = None
        for nd in range(self.nodes):
            g = dist.new_group(list(range(nd * node_size, (nd + 1) * node_size)))
            if nd == self.node:
                self.node_group = g
        self.cross_group = None
        for lr in range(node_size):
            g = dist.new_group(list(range(lr, self.world, node_size)))
            if lr == self.local:
                self.cross_group = g
        self.wslot = _slot_bytes(self.max_seg, wspec)
        self.gslot = _slot_bytes(self.max_seg, gspec)
        P = self.world
        dev = self.device
        self._ag_own = torch.zeros(self.wslot, dtype=torch.uint8, device=dev)
        self._ag_cross = torch.zeros(self.nodes * self.wslot, dtype=torch.uint8, device=dev)
        self._ag_all = torch.zeros(P * self.wslot, dtype=torch.uint8, device=dev)
        self._rs_send = torch.zeros(P * self.gslot, dtype=torch.uint8, device=dev)
        self._rs_mid = torch.zeros(P * self.gslot, dtype=torch.uint8, device=dev)
        self._rs_recv = torch.zeros(P * self.gslot, dtype=torch.uint8, device=dev)

    # -- slot views (a call's slots are sized by its largest segment) ------------------
    @staticmethod
    def _views(buf, ms, n, spec):
        cb, nb = codes_bytes(n, spec), num_buckets(n, spec.bucket)
        coff = (codes_bytes(ms, spec) + 255) // 256 * 256
        codes = buf[:max(cb, 1)]
        meta = buf[coff: coff + 12 * max(nb, 1)].view(torch.float32).view(max(nb, 1), 3)
        return codes[:cb], meta[:nb]

    # -- C1 ---------------------------------------------------------------------------
    def all_gather(self, shard: torch.Tensor, segs, key: SegmentKey, out: torch.Tensor) -> torch.Tensor:
        """``out`` (full tensor, element 0 = segs[0] start) receives every rank's
        dequantized shard; keys use worker 0 (sharded.py:341)."""
        P, spec = self.world, self.wspec
        s, n = segs[self.rank]
        if shard.numel() != n:
            raise ValueError("shard length does not match its segment")
        ms = max(m for _, m in segs)
        if ms > self.max_seg:
            raise ValueError("segment larger than the communicator's max_segment_elems")
        slot = _slot_bytes(ms, spec)
        own, cross, allb = self._ag_own[:slot], self._ag_cross[:self.nodes * slot], self._ag_all[:P * slot]
        if n:
            quantize_segments([(shard, s, SegmentKey(key.root_seed, key.step, key.layer, key.phase, 0))], spec,
                              out=[self._views(own, ms, n, spec)])
        # (1) across nodes: slot of (node j, my local index) for every node j
        dist.all_gather_into_tensor(cross, own, group=self.cross_group)
        # (2) inside the node: every local rank's cross-gathered slots -> [local][node] order
        dist.all_gather_into_tensor(allb, cross, group=self.node_group)
        jobs = []
        base = segs[0][0]
        for p in range(P):
            nd, lr = divmod(p, self.node_size)
            sp, np_ = segs[p]
            if np_ == 0:
                continue
            off = (lr * self.nodes + nd) * slot
            c, m = self._views(allb[off: off + slot], ms, np_, spec)
            jobs.append((c, m, np_, out[sp - base: sp - base + np_]))
        dequantize_segments(jobs, spec, out.dtype)
        return out

    # -- C2 ---------------------------------------------------------------------------
    def reduce_scatter(self, full_grad: torch.Tensor, segs, key: SegmentKey, out: torch.Tensor) -> torch.Tensor:
        """``out`` (this rank's shard) receives the fp64-ordered average of every
        rank's dequantized contribution (sharded.py:375-433); keys use worker = rank."""
        P, spec, L, N = self.world, self.gspec, self.node_size, self.nodes
        base = segs[0][0]
        ms = max(m for _, m in segs)
        if ms > self.max_seg:
            raise ValueError("segment larger than the communicator's max_segment_elems")
        slot = _slot_bytes(ms, spec)
        send, midb, recv = self._rs_send[:P * slot], self._rs_mid[:P * slot], self._rs_recv[:P * slot]
        k = SegmentKey(key.root_seed, key.step, key.layer, key.phase, self.rank)
        # send layout for the intra-node all-to-all: [dest local l][dest node j] slots
        items, outs = [], []
        for q in range(P):
            sq, nq = segs[q]
            if nq == 0:
                continue
            jq, lq = divmod(q, L)
            off = (lq * N + jq) * slot
            items.append((full_grad[sq - base: sq - base + nq], sq, k))
            outs.append(self._views(send[off: off + slot], ms, nq, spec))
        if items:
            quantize_segments(items, spec, out=outs)
        # (1) inside the node: local rank l receives [source local][dest node] slots for dest local l
        dist.all_to_all_single(midb, send, group=self.node_group)
        # regroup [src local][dest node] -> [dest node][src local] for the cross-node exchange
        mid = midb.view(L, N, slot).transpose(0, 1).contiguous().view(-1) if N > 1 and L > 1 else midb
        # (2) across nodes: dest node j receives [src node][src local] = sources in rank order
        dist.all_to_all_single(recv, mid, group=self.cross_group)
        s, n = segs[self.rank]
        if n == 0:
            return out
        sources = []
        for p in range(P):  # slot index = src node * L + src local = p
            off = p * slot
            sources.append(self._views(recv[off: off + slot], ms, n, spec))
        if P <= 8:
            dequant_accumulate(sources, n, spec, P, dtype=out.dtype, out=out)
        else:
            raise ValueError("at most 8 sources per K4 launch")
        return out
