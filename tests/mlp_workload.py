"""Test workload: the reference's toy sharded MLP training loop, with pluggable
collective hooks.

The step math restates ShardedMLP.train_step / forward_layer / backward_layer
(pkg/src/qsdp/sharded.py:437-503) and its data/parameter generators
(sharded.py:256-288), so that swapping only the two hooks reproduces the
reference run bit-for-bit:

* ``hooks="gpu"``    -- paper_2302_02390_b200.sharded.QSDPHooks (the product);
* ``hooks="oracle"`` -- the C oracle (test infrastructure, tests only).
"""

from __future__ import annotations

import math

import numpy as np

from paper_2302_02390_b200.sharded import (PHASE_GRAD, PHASE_W_BWD, PHASE_W_FWD, LayerSpec,
                                           LedgerEntry, QSDPHooks, QuantConfig, Transfer, shard_bounds)


def layer_specs(widths):
    out = []
    for i in range(len(widths) - 1):
        out.append(LayerSpec(f"dense{i}", "dense", (widths[i], widths[i + 1])))
        out.append(LayerSpec(f"bias{i}", "bias", (widths[i + 1],)))
    return out


def init_params(widths, param_seed):
    g = np.random.default_rng(np.random.SeedSequence((param_seed, 0)))
    p = {}
    for i in range(len(widths) - 1):
        p[f"dense{i}"] = g.standard_normal(widths[i] * widths[i + 1]) / math.sqrt(widths[i])
        p[f"bias{i}"] = 0.01 * g.standard_normal(widths[i + 1])
    return p


def batch_for(widths, batch, data_seed, step):
    teacher = np.random.default_rng(np.random.SeedSequence((data_seed, 1))).standard_normal(
        (widths[0], widths[-1])) / math.sqrt(widths[0])
    x = np.random.default_rng(np.random.SeedSequence((data_seed, 2, step))).standard_normal(
        (batch, widths[0]))
    return x, x @ teacher


class _Cfg:
    def __init__(self, P, root_seed):
        self.P = P
        self.root_seed = root_seed


class _Model:
    def __init__(self, params, layers, P):
        self.bounds, self.shards = {}, {}
        for layer in layers:
            flat = np.asarray(params[layer.name], dtype=float).ravel()
            b = shard_bounds(flat.size, P)
            self.bounds[layer.name] = b
            self.shards[layer.name] = [flat[s:e].copy() for s, e in b]

    def full(self, name):
        return np.concatenate(self.shards[name])


class _OracleHooks:
    """The same hooks evaluated by the C oracle (tests only)."""

    def _gather(self, step, layer_idx, phase, entry):
        from oracle import oracle as O
        layer = self.layers[layer_idx]
        P, q = self.cfg.P, self.quant
        full = self.model.full(layer.name)
        bounds = self.model.bounds[layer.name]
        if layer.kind == "dense" and q.quantize_weights:
            out = O.gather(full, P, q.bucket_size, q.weight_bits, self.cfg.root_seed, step, layer_idx, phase)
            for s, e in bounds:
                if e > s:
                    entry.record(Transfer("allgather", layer.name, q.weight_bits,
                                          O.message_size_bits(e - s, q.bucket_size, q.weight_bits) // 8,
                                          P - 1, (e - s) * q.weight_bits))
        else:
            out = full.copy()
            w = q.raw_bits if layer.kind == "dense" else 32
            for s, e in bounds:
                if e > s:
                    entry.record(Transfer("allgather", layer.name, w, (e - s) * w // 8, P - 1, (e - s) * w))
        entry.allgather_events += 1
        return out

    def _reduce_scatter(self, step, layer_idx, grads, entry):
        from oracle import oracle as O
        layer = self.layers[layer_idx]
        P, q = self.cfg.P, self.quant
        bounds = self.model.bounds[layer.name]
        quantized = layer.kind == "dense" and q.quantize_gradients
        if quantized:
            outs = O.reduce_scatter(grads, q.bucket_size, q.gradient_bits, self.cfg.root_seed, step, layer_idx)
        else:
            outs = []
            for s, e in bounds:
                acc = np.zeros(e - s)
                for p in range(P):
                    acc = acc + np.asarray(grads[p])[s:e]
                outs.append(acc / P)
        for qq, (s, e) in enumerate(bounds):
            if e == s:
                continue
            for p in range(P):
                if p == qq:
                    continue
                if quantized:
                    entry.record(Transfer("reducescatter", layer.name, q.gradient_bits,
                                          O.message_size_bits(e - s, q.bucket_size, q.gradient_bits) // 8,
                                          1, (e - s) * q.gradient_bits))
                else:
                    w = q.raw_gradient_bits if layer.kind == "dense" else 32
                    entry.record(Transfer("reducescatter", layer.name, w, (e - s) * w // 8, 1, (e - s) * w))
        entry.reducescatter_events += 1
        return outs


class _Base:
    def __init__(self, widths, P, batch, lr, quant: QuantConfig, seed=0):
        self.widths = list(widths)
        self.cfg = _Cfg(P, seed)
        self.batch, self.lr, self.quant = batch, lr, quant
        self.seed = seed
        self.layers = layer_specs(self.widths)
        self.model = _Model(init_params(self.widths, seed), self.layers, P)
        self.pairs = len(self.widths) - 1

    def train_step(self, step):
        P = self.cfg.P
        entry = LedgerEntry(step=step)
        x, y = batch_for(self.widths, self.batch, self.seed, step)
        rows = self.batch // P
        xs = [x[p * rows:(p + 1) * rows] for p in range(P)]
        ys = [y[p * rows:(p + 1) * rows] for p in range(P)]
        inputs, outputs, hs = [], [], xs
        for i in range(self.pairs):
            inputs.append(hs)
            w = self._gather(step, 2 * i, PHASE_W_FWD, entry).reshape(self.layers[2 * i].shape)
            b = self._gather(step, 2 * i + 1, PHASE_W_FWD, entry)
            zs = [h @ w + b for h in hs]
            hs = zs if i == self.pairs - 1 else [np.tanh(z) for z in zs]
            outputs.append(hs)
        losses = [float(((hs[p] - ys[p]) ** 2).sum() / (2 * rows)) for p in range(P)]
        dzs = [(hs[p] - ys[p]) / rows for p in range(P)]
        for i in range(self.pairs - 1, -1, -1):
            w = self._gather(step, 2 * i, PHASE_W_BWD, entry).reshape(self.layers[2 * i].shape)
            self._gather(step, 2 * i + 1, PHASE_W_BWD, entry)
            dw = [(inputs[i][p].T @ dzs[p]).ravel() for p in range(P)]
            db = [dzs[p].sum(axis=0) for p in range(P)]
            prev = None
            if i > 0:
                prev = [(dzs[p] @ w.T) * (1.0 - outputs[i - 1][p] ** 2) for p in range(P)]
            aw = self._reduce_scatter(step, 2 * i, dw, entry)
            ab = self._reduce_scatter(step, 2 * i + 1, db, entry)
            for q in range(P):
                self.model.shards[f"dense{i}"][q] -= self.lr * aw[q]
                self.model.shards[f"bias{i}"][q] -= self.lr * ab[q]
            dzs = prev
        return float(np.mean(losses)), entry

    def full_params(self):
        return {layer.name: self.model.full(layer.name) for layer in self.layers}


class GpuMLP(QSDPHooks, _Base):
    pass


class OracleMLP(_OracleHooks, _Base):
    pass


def make(hooks, **kw):
    return (GpuMLP if hooks == "gpu" else OracleMLP)(**kw)
