"""Generate golden vectors from the LIVE reference (run in the dev container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/golden.npz.  Every array is produced by the unmodified
reference functions:

* noise:    np.random.SeedSequence(key).generate_state(4, uint64) and the first
            draws of bucket_rng(*key) (pkg/src/qsdp/sharded.py:235-240);
* quant_*:  _segment_blocks(...) -> QuantizedBlock codes/scales/shift, encode()
            wire bytes, dequantize() fp64 (quantize.py:209-286, wire.py:108-131,
            sharded.py:243-248);
* lv_*:     inner="levels" (quantize.py:235-286, 400-422) codes/scales and
            dequantize(block, "levels", table) (quantize.py:225-231) over
            uniform, learned, out-of-[0,1] and 2^12 / 2^16-level tables;
* ll_*:     learn_levels(values, table, lr) outputs (quantize.py:366-397),
            including the re-sort / collision-nudge and distinct-count paths;
* wire_*:   malformed / edge-case messages and the exception class (or "ok") the
            reference decode() raises for each (wire.py:134-184);
* lat_*:    the lattice-projected step fused with the RS epilogue
            (optimizer.py:194-229): the reduce-scatter average of P ranks'
            quantized gradients (sharded.py:375-433 pipeline), then the
            reference's qsdp_step with that gradient and the keyed shift
            r = sample_shift(d, bucket_rng(root, step, layer, 3, 0, 0));
* ledger_csv: CommLedger.to_csv bytes of a ShardedMLP run (sharded.py:161-181);
* hook_*:   inputs/outputs of ShardedMLP._gather / ._reduce_scatter recorded
            during a short ShardedMLP run (sharded.py:323-433), plus the run's
            ledger bits and losses, and ReferenceMLP's final parameters.

The fixtures travel to the GPU box (the reference does not); tests compare both
the C oracle and the CUDA path against them.
"""

from __future__ import annotations

import os
import sys

import numpy as np

from qsdp.quantize import BucketSpec, LevelTable, bucketed_quantize, dequantize, learn_levels
from qsdp.sharded import (
    PHASE_GRAD,
    QuantConfig,
    ReferenceMLP,
    ShardedMLP,
    SimConfig,
    _segment_blocks,
    bucket_rng,
)
from qsdp.wire import _pack_codes, encode

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def _cases():
    """(bits, inner, bucket, n, start, key, dtype, distribution) quantizer cases."""
    rng = np.random.default_rng(20230205)
    cases = []
    # The paper's configurations: w8 shift / g8, g4 stochastic, bucket 1024.
    for bits, inner in [(8, "shift"), (8, "uniform_stochastic"), (4, "uniform_stochastic"),
                        (4, "shift"), (6, "shift"), (5, "uniform_stochastic")]:
        cases.append((bits, inner, 1024, 3000, 4096, (0, 3, 2, 0 if inner == "shift" else 2, 1),
                      "f32", "normal"))
    # bucket-size sweep 64..4096 (350M config), short last buckets, odd starts
    for S in (64, 128, 256, 512, 2048, 4096):
        cases.append((4, "uniform_stochastic", S, 5 * S + 17, 123457, (7, 1, 4, 2, 3), "f32", "normal"))
        cases.append((8, "shift", S, 3 * S + 5, 999, (7, 1, 4, 1, 0), "f32", "normal"))
    # every bit width 1..16, both modes, fp64 inputs (the reference's dtype)
    for bits in range(1, 17):
        for inner in ("shift", "uniform_stochastic"):
            cases.append((bits, inner, 100, 333, int(rng.integers(0, 2**31)),
                          (1, 2, 3, 0 if inner == "shift" else 2, 0), "f64", "normal"))
    # stress: heavy tails, constant (degenerate) buckets, tiny ranges, large keys
    cases.append((8, "shift", 1024, 4096, 0, (0, 0, 0, 0, 0), "f32", "student_t"))
    cases.append((8, "uniform_stochastic", 1024, 4096, 0, (0, 0, 0, 2, 5), "f32", "constant_mix"))
    cases.append((8, "shift", 1024, 2500, 2**33 + 5, (2**40 + 3, 2**35, 1, 0, 0), "f32", "tiny"))
    cases.append((16, "uniform_stochastic", 1024, 2048, 77, (5, 9, 11, 2, 7), "f64", "normal"))
    cases.append((8, "shift", 7, 50, 3, (1, 1, 1, 1, 0), "f64", "ties"))
    return cases


def _input(n, dtype, dist, rng):
    if dist == "normal":
        x = rng.standard_normal(n) * 0.02
    elif dist == "student_t":
        x = rng.standard_t(3, n) * 0.02
    elif dist == "constant_mix":
        x = rng.standard_normal(n) * 1e-3
        x[1024:2048] = 0.25          # one fully degenerate bucket
        x[3072:4096] = -0.0          # zeros
    elif dist == "tiny":
        x = (rng.standard_normal(n) * 1e-36)
    elif dist == "ties":
        x = np.tile(np.array([0.0, 0.5, 1.0, 1.5, 2.0, 2.5, 3.0]), n // 7 + 1)[:n]
    else:
        raise ValueError(dist)
    if dtype == "f32":
        x = x.astype(np.float32).astype(np.float64)
    return x


def _level_tables(rng):
    """(name, levels) tables for the levels-mode cases."""
    tabs = [LevelTable.uniform(b).levels for b in (1, 2, 3, 4, 8)]
    g = rng.standard_normal(20000)
    g = (g - g.min()) / (g.max() - g.min())
    for b, lr, passes in ((2, 0.01, 1), (3, 0.05, 2), (4, 0.01, 1), (8, 0.01, 1)):
        t = LevelTable.uniform(b)
        for _ in range(passes):
            t = learn_levels(g, t, lr)
        tabs.append(t.levels)
    tabs.append(np.array([-0.5, 0.1, 0.2, 1.7]))                       # levels outside [0, 1]
    tabs.append(np.array([0.0, 0.5, np.nextafter(0.5, 1.0), 1.0]))      # mid rounds onto a level
    tabs.append(np.sort(rng.uniform(0, 1, 1 << 12)))                    # smem-staged widest
    tabs.append(np.linspace(0.0, 1.0, 1 << 16) + rng.uniform(-1e-7, 1e-7, 1 << 16))  # global mids
    return tabs


def _levels(out):
    rng = np.random.default_rng(402)
    tabs = _level_tables(rng)
    rows = []
    for i, q in enumerate(tabs):
        table = LevelTable(q)
        bits = table.bit_width
        out[f"lvtab_{i}"] = table.levels
        for j, (S, n, dist, dtype) in enumerate([(1024, 3000, "normal", "f32"), (100, 333, "normal", "f64"),
                                                 (7, 50, "ties", "f64"), (64, 640, "mids", "f64")]):
            if dist == "mids":   # values landing exactly on the table's mids (lo=0, hi=1 buckets)
                mids = (table.levels[:-1] + table.levels[1:]) / 2
                x = np.resize(np.concatenate([[0.0, 1.0], np.clip(mids, 0, 1),
                                              np.nextafter(np.clip(mids, 0, 1), 2)]), n)
                for b0 in range(0, n, S):
                    x[b0], x[b0 + 1] = 0.0, 1.0
            else:
                x = _input(n, dtype, dist, rng)
            blocks = bucketed_quantize(x, BucketSpec(S), bits, "levels", levels=table)
            k = len(rows)
            out[f"lv_{k}_x"] = x.astype(np.float32) if dtype == "f32" else x
            out[f"lv_{k}_codes"] = np.frombuffer(b"".join(_pack_codes(b.codes, bits) for b in blocks),
                                                 dtype=np.uint8)
            out[f"lv_{k}_meta"] = np.array([[b.shift, b.scale_lo, b.scale_hi] for b in blocks],
                                           dtype=np.float32)
            out[f"lv_{k}_deq"] = np.concatenate([dequantize(b, "levels", table) for b in blocks])
            rows.append([i, bits, S, n])
    out["lv_cases"] = np.array(rows, dtype=np.int64)
    # learn_levels
    lrows = []
    g = rng.standard_normal(50000)
    g = (g - g.min()) / (g.max() - g.min())
    lcases = [(g[:5000], LevelTable.uniform(2).levels, 0.01), (g, LevelTable.uniform(4).levels, 0.01),
              (g[:20000], LevelTable.uniform(8).levels, 0.05), (rng.uniform(0, 1, 3000), LevelTable.uniform(3).levels, 0.2),
              (np.array([0.375, 0.9, 0.95, 0.99]), np.array([0.0, 0.25, 0.5, 1.0]), 2.0),   # collision -> nudge
              (np.array([0.404, 0.1, 0.7, 0.2]), np.array([0.0, 0.4, 0.41, 1.0]), 3.0),    # crossing -> re-sort
              (np.array([0.3, 0.3, 0.6]), LevelTable.uniform(2).levels, 0.1)]              # too few distinct
    import warnings
    for k, (v, q0, lr) in enumerate(lcases):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", RuntimeWarning)
            res = learn_levels(v, LevelTable(q0), lr).levels
        out[f"ll_{k}_values"] = np.asarray(v, dtype=np.float64)
        out[f"ll_{k}_init"] = np.asarray(q0, dtype=np.float64)
        out[f"ll_{k}_out"] = res
        lrows.append(lr)
    out["ll_lr"] = np.array(lrows)


def _lattice_cases(out):
    from qsdp.optimizer import RunPlan, qsdp_step
    from qsdp.quantize import sample_shift
    rng = np.random.default_rng(733)

    class _Stub:  # a "problem" whose stochastic gradient is the reduce-scatter average
        def __init__(self, g, beta):
            self.g, self.smoothness = g, beta

        def stochastic_gradient(self, x, rng):
            return self.g

        def objective(self, x):
            return 0.0

    rows = []
    for k, (P, bits, S, n, eta, beta, dstar, ratio) in enumerate(
            [(2, 8, 1024, 5000, 0.5, 2.0, 0.01, 64), (4, 4, 256, 3001, 0.3, 1.0, 0.001, 16),
             (3, 8, 100, 777, 1.0, 4.0, 1e-4, 3), (1, 6, 64, 640, 0.25, 1.5, 0.05, 128)]):
        root, step, layer = 5, 7 + k, 2
        grads = [(rng.standard_normal(n) * 1e-2).astype(np.float32).astype(np.float64) for _ in range(P)]
        acc = np.zeros(n)
        for p in range(P):
            blocks = _segment_blocks(grads[p], 0, S, bits, "uniform_stochastic",
                                     lambda st, p=p: bucket_rng(root, step, layer, PHASE_GRAD, p, st))
            acc = acc + np.concatenate([dequantize(b, "uniform_stochastic") for b in blocks])
        ghat = acc / P
        d = dstar / ratio
        plan = RunPlan(eta=eta, coarse_resolution=dstar, fine_resolution=d, iteration_count=1, epsilon=1.0,
                       grid_ratio=ratio)
        r = sample_shift(d, bucket_rng(root, step, layer, 3, 0, 0))
        x = rng.standard_normal(n) * 0.1
        x_new, rec = qsdp_step(x, _Stub(ghat, beta), plan, rng, shift=r)
        assert rec.shift == r
        out[f"lat_{k}_grads"] = np.stack(grads).astype(np.float32)
        out[f"lat_{k}_x"] = x
        out[f"lat_{k}_ghat"] = ghat
        out[f"lat_{k}_xnew"] = x_new
        out[f"lat_{k}_r"] = np.array(r)
        rows.append([P, bits, S, n, root, step, layer, eta, beta, d])
    out["lat_cases"] = np.array(rows, dtype=np.float64)


def _wire_cases(out):
    from qsdp.quantize import QuantizedBlock
    from qsdp.wire import decode
    import struct
    rng = np.random.default_rng(611)

    def blk(codes, bits, shift=0.0, lo=0.0, hi=1.0):
        c = np.asarray(codes, dtype=np.uint32)
        return QuantizedBlock(codes=c, shift=shift, scale_lo=lo, scale_hi=hi, bit_width=bits, length=c.size)

    base = encode([blk(rng.integers(0, 8, 5), 3), blk(rng.integers(0, 8, 5), 3), blk(rng.integers(0, 8, 3), 3)])
    two = encode([blk(np.arange(4), 4), blk(np.arange(4), 4)])
    msgs = [b"", b"\x01\x02", base, base[:13], base[:14], base[:20], base[:14 + 12], base[:14 + 13 + 1],
            base[:-1], base + b"\x00", base + b"\x00\x00\x07"]
    m = bytearray(base); m[0] = 9; msgs.append(bytes(m))
    m = bytearray(base); m[1] = 0; msgs.append(bytes(m))
    m = bytearray(base); m[1] = 40; msgs.append(bytes(m))
    m = bytearray(base); m[1] = 17; msgs.append(bytes(m))
    m = bytearray(two); m[10:14] = (99).to_bytes(4, "little"); msgs.append(bytes(m))
    m = bytearray(two); m[2:6] = (0).to_bytes(4, "little"); msgs.append(bytes(m))
    m = bytearray(base); m[14 + 12 + 1] ^= 0x80; msgs.append(bytes(m))            # padding bit of block 0
    m = bytearray(base); m[-1] ^= 0x40; msgs.append(bytes(m))                     # padding of the last block
    m = bytearray(base); m[14 + 4:14 + 8] = struct.pack("<f", 5.0); msgs.append(bytes(m))  # lo > hi, block 0
    m = bytearray(base); m[14 + 14 + 4:14 + 14 + 8] = struct.pack("<f", float("nan")); msgs.append(bytes(m))
    m = bytearray(base); m[14 + 14 + 4:14 + 14 + 8] = struct.pack("<f", 5.0); m[-1] ^= 0x40; msgs.append(bytes(m))
    m = bytearray(base); m[-1] ^= 0x40; msgs.append(bytes(m[:-2]))               # padding + truncation later
    m = bytearray(base); m[14 + 12 + 1] ^= 0x80; msgs.append(bytes(m[:-1]))      # padding at 0, truncated at 2
    msgs.append(bytes([1, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0]))                  # canonical empty
    msgs.append(bytes([1, 0, 0, 0, 0, 0, 0, 0, 0, 0, 5, 0, 0, 0]))                  # empty with total 5
    msgs.append(bytes([1, 3, 5, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0]) + b"\x00")       # empty + trailing
    for i, msg in enumerate(msgs):
        try:
            decode(msg)
            res = "ok"
        except Exception as e:  # noqa: BLE001 - record the class
            res = type(e).__name__
        out[f"wire_{i}_msg"] = np.frombuffer(msg, dtype=np.uint8) if msg else np.zeros(0, dtype=np.uint8)
        out[f"wire_{i}_res"] = np.array(res)
    out["wire_n"] = np.array(len(msgs))


def main():
    rng = np.random.default_rng(7)
    out = {"numpy_version": np.array(np.__version__)}

    # ---- noise -------------------------------------------------------------
    keys = []
    for k in range(64):
        key = [int(v) for v in rng.integers(0, 2**31, 6)]
        if k % 4 == 1:
            key[5] = int(rng.integers(2**32, 2**40))     # start >= 2**32 (two words)
        if k % 4 == 2:
            key[0] = int(rng.integers(2**32, 2**62))     # large root seed
        if k % 8 == 3:
            key = [0, 0, 0, 0, 0, 0]
        keys.append(key)
    keys = np.array(keys, dtype=np.uint64)
    states = np.stack([np.random.SeedSequence(tuple(int(v) for v in k)).generate_state(4, np.uint64)
                       for k in keys])
    draws = np.stack([bucket_rng(*[int(v) for v in k]).bit_generator.random_raw(8) for k in keys])
    out.update(noise_keys=keys, noise_states=states, noise_draws=np.asarray(draws, dtype=np.uint64))

    # ---- quantizer ---------------------------------------------------------
    cases = _cases()
    meta_rows = []
    for i, (bits, inner, S, n, start, key, dtype, dist) in enumerate(cases):
        x = _input(n, dtype, dist, rng)
        blocks = _segment_blocks(x, start, S, bits, inner, lambda s: bucket_rng(*key, s))
        codes = b"".join(_pack_codes(b.codes, bits) for b in blocks)
        meta = np.array([[b.shift, b.scale_lo, b.scale_hi] for b in blocks], dtype=np.float32)
        deq = np.concatenate([dequantize(b, inner) for b in blocks])
        out[f"quant_{i}_x"] = x.astype(np.float32) if dtype == "f32" else x
        out[f"quant_{i}_codes"] = np.frombuffer(codes, dtype=np.uint8)
        out[f"quant_{i}_meta"] = meta
        out[f"quant_{i}_deq"] = deq
        out[f"quant_{i}_wire"] = np.frombuffer(encode(blocks), dtype=np.uint8)
        meta_rows.append([bits, 0 if inner == "shift" else 1, S, n, start, *key])
    out["quant_cases"] = np.array(meta_rows, dtype=np.int64)

    # ---- protocol hooks: record a short ShardedMLP run ------------------------
    hook_rows = []
    hook_idx = 0
    for P, quant in [(4, QuantConfig()), (2, QuantConfig(gradient_bits=4, bucket_size=64)),
                     (3, QuantConfig(weight_bits=6, bucket_size=100))]:
        cfg = SimConfig(widths=(64, 64, 10), P=P, batch=24, lr=0.05, quant=quant,
                        root_seed=11, param_seed=11, data_seed=11)
        sim = ShardedMLP(cfg)
        rec = []
        orig_g, orig_rs = sim._gather, sim._reduce_scatter

        def g(step, layer_idx, phase, entry, _o=orig_g, _rec=rec, _sim=sim):
            layer = _sim.layers[layer_idx]
            shards = [s.copy() for s in _sim.model.shards[layer.name]]
            res = _o(step, layer_idx, phase, entry)
            _rec.append(("ag", step, layer_idx, phase, layer.kind, shards, res))
            return res

        def rs(step, layer_idx, grads, entry, _o=orig_rs, _rec=rec, _sim=sim):
            layer = _sim.layers[layer_idx]
            res = _o(step, layer_idx, grads, entry)
            _rec.append(("rs", step, layer_idx, PHASE_GRAD, layer.kind,
                         [np.asarray(gg).copy() for gg in grads], res))
            return res

        sim._gather, sim._reduce_scatter = g, rs
        losses, bits_ag, bits_rs = [], [], []
        for t in range(2):
            loss, entry = sim.train_step(t)
            losses.append(loss)
            bits_ag.append(entry.allgather_bits)
            bits_rs.append(entry.reducescatter_bits)
        if not hook_rows:
            import tempfile
            with tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False) as fh:
                path = fh.name
            sim.ledger.to_csv(path)
            out["ledger_csv"] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)
            os.unlink(path)
        ref = ReferenceMLP(cfg)
        ref_losses = ref.run(2)
        assert ref_losses == losses
        run_id = len(hook_rows)
        for kind, step, li, phase, lkind, ins, res in rec:
            if lkind != "dense":
                continue   # exempt layers are raw copies; covered by host tests
            out[f"hook_{hook_idx}_in"] = np.stack([np.asarray(v) for v in ins]) if kind == "rs" \
                else np.concatenate(ins)
            out[f"hook_{hook_idx}_out"] = np.concatenate(res) if kind == "rs" else res
            out[f"hookmeta_{hook_idx}"] = np.array(
                [run_id, 0 if kind == "ag" else 1, step, li, phase], dtype=np.int64)
            hook_idx += 1
        out[f"run_{run_id}_cfg"] = np.array(
            [P, quant.weight_bits, quant.gradient_bits, quant.bucket_size, 11], dtype=np.int64)
        out[f"run_{run_id}_losses"] = np.array(losses)
        out[f"run_{run_id}_bits"] = np.array([bits_ag, bits_rs], dtype=np.int64)
        for name, v in ref.params.items():
            out[f"run_{run_id}_param_{name}"] = v
        hook_rows.append(run_id)
    out["n_hooks"] = np.array(hook_idx)
    _levels(out)
    _wire_cases(out)
    _lattice_cases(out)
    out["n_runs"] = np.array(len(hook_rows))
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT}: {os.path.getsize(OUT)/1e6:.2f} MB, {len(cases)} quant cases, "
          f"{hook_idx} hook calls")


if __name__ == "__main__":
    sys.exit(main())
