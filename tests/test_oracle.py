"""CPU: pin the C oracle against the reference's golden vectors, its own
known-answer tests, and (when mounted) the live reference."""

import os

import numpy as np
import pytest

from conftest import golden_cases, golden_hooks


def test_noise_matches_numpy_golden(golden, oracle):
    for key, state, draws in zip(golden["noise_keys"], golden["noise_states"], golden["noise_draws"]):
        key = [int(v) for v in key]
        assert np.array_equal(oracle.seedseq_state(key), state)
        g = oracle.PCG64(*key)
        assert [g.next_raw() for _ in range(len(draws))] == [int(d) for d in draws]


def test_quantizer_golden(golden, oracle):
    for c in golden_cases(golden):
        x = c["x"].astype(np.float64)
        codes, meta, bad = oracle.quantize_segment(x, c["start"], c["bucket"], c["bits"], c["inner"], c["key"])
        assert bad == -1
        assert np.array_equal(codes, c["codes"]), c["i"]
        assert np.array_equal(meta, c["meta"]), c["i"]          # == semantics (QuantizedBlock.__eq__)
        deq = oracle.dequantize_segment(codes, meta, c["n"], c["bucket"], c["bits"])
        assert np.array_equal(deq, c["deq"]), c["i"]
        assert oracle.encode_segment(codes, meta, c["n"], c["bucket"], c["bits"]) == c["wire"].tobytes()
        assert oracle.message_size_bits(c["n"], c["bucket"], c["bits"]) == 8 * c["wire"].size


def test_oracle_threads_do_not_change_results(golden, oracle):
    for c in list(golden_cases(golden))[:8]:
        a = oracle.quantize_segment(c["x"], c["start"], c["bucket"], c["bits"], c["inner"], c["key"], 1)
        b = oracle.quantize_segment(c["x"], c["start"], c["bucket"], c["bits"], c["inner"], c["key"], 4)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_hook_replays_golden(golden, oracle):
    """ShardedMLP._gather/_reduce_scatter outputs recorded from the reference."""
    for h in golden_hooks(golden):
        if h["kind"] == "ag":
            out = oracle.gather(h["inp"], h["P"], h["bucket"], h["wbits"], h["seed"], h["step"], h["layer"],
                                h["phase"])
        else:
            out = np.concatenate(oracle.reduce_scatter(list(h["inp"]), h["bucket"], h["gbits"], h["seed"],
                                                       h["step"], h["layer"]))
        assert np.array_equal(out, h["out"]), h


# --- reference KATs (pkg/tests/test_quantize.py, test_wire.py) restated on the oracle ---

def test_kat_ties_to_even(oracle):
    # test_quantize.py:48-51 -- np.round half to even on the unshifted grid is exercised
    # through the "ties" golden case; here: bucket of [0, 1] at b=1 never produces code > 1.
    c, m, _ = oracle.quantize_segment(np.array([0.0, 1.0]), 0, 2, 1, 0, (0, 0, 0, 0, 0))
    assert oracle.unpack(c, 2, 1).max() <= 1


def test_kat_stochastic_on_level(oracle):
    # test_quantize.py:291-295: values exactly on levels keep their code.
    x = np.array([0.0, 1 / 15, 1.0])
    c, m, _ = oracle.quantize_segment(x, 0, 3, 4, 1, (0, 0, 0, 2, 0))
    assert list(oracle.unpack(c, 3, 4)) == [0, 1, 15]


def test_kat_constant_bucket_roundtrips(oracle):
    # test_quantize.py:229-234
    x = np.full(100, 0.3)
    c, m, _ = oracle.quantize_segment(x, 0, 1024, 8, 0, (0, 0, 0, 0, 0))
    assert m[0, 0] == 0.0 and m[0, 1] == m[0, 2]
    assert np.all(oracle.dequantize_segment(c, m, 100, 1024, 8) == np.float32(0.3))


def test_kat_wire_sizes(oracle):
    # test_wire.py:50-69
    assert oracle.codes_bytes(8, 8, 4) == 4
    assert oracle.codes_bytes(3, 3, 3) == 2
    assert oracle.message_size_bits(1024, 1024, 8) == 8192 + 96 + 112
    assert oracle.message_size_bits(0, 1024, 8) == 112


def test_kat_nonfinite_index(oracle):
    x = np.zeros(3000)
    x[2500] = np.nan
    _, _, bad = oracle.quantize_segment(x, 0, 1024, 8, 0, (0, 0, 0, 0, 0))
    assert bad == 2500


# --- live reference ---------------------------------------------------------------

@pytest.mark.reference
def test_live_reference_random(oracle, reference):
    from qsdp.quantize import dequantize
    from qsdp.sharded import _segment_blocks, bucket_rng
    from qsdp.wire import encode
    rng = np.random.default_rng(123)
    for trial in range(40):
        bits = int(rng.integers(1, 17))
        inner = int(rng.integers(0, 2))
        S = int(rng.choice([8, 64, 100, 256, 1024]))
        n = int(rng.integers(1, 2500))
        x = rng.standard_normal(n) * 10.0 ** rng.uniform(-6, 3)
        if trial % 2:
            x = x.astype(np.float32).astype(np.float64)
        key = tuple(int(v) for v in rng.integers(0, 2**33, 5))
        start = int(rng.integers(0, 2**34))
        mode = "uniform_stochastic" if inner else "shift"
        blocks = _segment_blocks(x, start, S, bits, mode, lambda s: bucket_rng(*key, s))
        codes, meta, _ = oracle.quantize_segment(x, start, S, bits, inner, key)
        assert oracle.encode_segment(codes, meta, n, S, bits) == encode(blocks)
        ref = np.concatenate([dequantize(b, mode) for b in blocks])
        assert np.array_equal(oracle.dequantize_segment(codes, meta, n, S, bits), ref)


@pytest.mark.reference
@pytest.mark.parametrize("P", [1, 2, 4])
def test_oracle_mlp_matches_reference_mlp(P, reference):
    """Acceptance criterion 7 (test_acceptance.py:258-290) with the oracle's hooks."""
    from qsdp.sharded import QuantConfig as RQ, ReferenceMLP, SimConfig

    import mlp_workload as W
    from paper_2302_02390_b200.sharded import QuantConfig
    ref = ReferenceMLP(SimConfig(widths=(64, 64, 10), P=P, batch=32, lr=0.05, quant=RQ(),
                                 root_seed=0, param_seed=0, data_seed=0))
    sim = W.make("oracle", widths=(64, 64, 10), P=P, batch=32, lr=0.05, quant=QuantConfig(), seed=0)
    for t in range(6):
        assert sim.train_step(t)[0] == ref.train_step(t)
    for name, full in sim.full_params().items():
        assert np.array_equal(full, ref.params[name])


def test_oracle_mlp_matches_golden_run(golden):
    import mlp_workload as W
    from paper_2302_02390_b200.sharded import QuantConfig
    for run in range(int(golden["n_runs"])):
        P, wb, gb, S, seed = (int(v) for v in golden[f"run_{run}_cfg"])
        sim = W.make("oracle", widths=(64, 64, 10), P=P, batch=24, lr=0.05,
                     quant=QuantConfig(weight_bits=wb, gradient_bits=gb, bucket_size=S), seed=seed)
        losses, ag, rs = [], [], []
        for t in range(len(golden[f"run_{run}_losses"])):
            loss, e = sim.train_step(t)
            losses.append(loss)
            ag.append(e.allgather_bits)
            rs.append(e.reducescatter_bits)
        assert np.allclose(losses, golden[f"run_{run}_losses"], rtol=1e-12, atol=0)
        assert ag == list(golden[f"run_{run}_bits"][0]) and rs == list(golden[f"run_{run}_bits"][1])


# -- learned levels -------------------------------------------


def test_levels_quantizer_golden(golden, oracle):
    from conftest import golden_level_cases
    n = 0
    for c in golden_level_cases(golden):
        codes, meta, bad = oracle.quantize_levels_segment(c["x"].astype(np.float64), c["bucket"], c["bits"],
                                                          c["table"])
        assert bad == -1
        np.testing.assert_array_equal(codes, c["codes"], err_msg=f"levels case {c['k']}")
        np.testing.assert_array_equal(meta, c["meta"])
        deq = oracle.dequantize_levels_segment(codes, meta, c["n"], c["bucket"], c["bits"], c["table"])
        np.testing.assert_array_equal(deq, c["deq"])
        n += 1
    assert n >= 40


def test_learn_levels_golden(golden, oracle):
    from conftest import golden_learn_cases
    for c in golden_learn_cases(golden):
        out = oracle.learn_levels(c["values"], c["init"], c["lr"])
        np.testing.assert_array_equal(out, c["out"], err_msg=f"learn case {c['k']}")


def test_kat_quantize_with_levels(oracle):
    # reference test_quantize.py: quantize_with_levels([0, .2, .7, 1], uniform(2)) == [0, 1, 2, 3]
    q = np.linspace(0.0, 1.0, 4)
    np.testing.assert_array_equal(oracle.level_codes([0.0, 0.2, 0.7, 1.0], q), [0, 1, 2, 3])
    # searchsorted side="left": a value exactly on a mid takes the lower level
    mids = (q[:-1] + q[1:]) / 2
    np.testing.assert_array_equal(oracle.level_codes(mids, q), [0, 1, 2])
    np.testing.assert_array_equal(oracle.level_codes(np.nextafter(mids, 2.0), q), [1, 2, 3])
    # out-of-span values clamp to the end levels
    np.testing.assert_array_equal(oracle.level_codes([-3.0, 7.0], q), [0, 3])


@pytest.mark.reference
def test_levels_live_reference_random(oracle, reference):
    from qsdp.quantize import BucketSpec, LevelTable, bucketed_quantize, learn_levels
    from qsdp.wire import _pack_codes
    rng = np.random.default_rng(5)
    for trial in range(6):
        bits = int(rng.integers(1, 7))
        g = rng.standard_normal(4000)
        g = (g - g.min()) / (g.max() - g.min())
        lr = float(rng.uniform(0.001, 0.1))
        table = learn_levels(g, LevelTable.uniform(bits), lr)
        np.testing.assert_array_equal(oracle.learn_levels(g, LevelTable.uniform(bits).levels, lr), table.levels)
        S = int(rng.integers(5, 300))
        x = rng.standard_normal(int(rng.integers(1, 2000)))
        blocks = bucketed_quantize(x, BucketSpec(S), bits, "levels", levels=table)
        codes, meta, _ = oracle.quantize_levels_segment(x, S, bits, table.levels)
        assert codes.tobytes() == b"".join(_pack_codes(b.codes, bits) for b in blocks)


# -- counter-based noise (numpy Philox4x64-10 keyed like bucket_rng) --------------------


def test_philox_draws_match_numpy_golden(golden_philox, oracle):
    for key, draws in zip(golden_philox["ph_keys"], golden_philox["ph_draws"]):
        g = oracle.Philox(*(int(k) for k in key))
        assert [g.next_raw() for _ in range(draws.size)] == [int(d) for d in draws]


def test_philox_quantizer_golden(golden_philox, oracle):
    from conftest import golden_philox_cases
    for c in golden_philox_cases(golden_philox):
        codes, meta, bad = oracle.quantize_segment(c["x"], c["start"], c["bucket"], c["bits"], c["inner"], c["key"],
                                                   4, noise=1)
        assert bad == -1
        assert np.array_equal(codes, c["codes"]), c["i"]
        assert np.array_equal(meta, c["meta"]), c["i"]
        assert np.array_equal(oracle.dequantize_segment(codes, meta, c["n"], c["bucket"], c["bits"]), c["deq"]), c["i"]


@pytest.mark.reference
def test_philox_live_reference_random(oracle, reference):
    """quantize_bucket(v, b, inner, Generator(Philox(SeedSequence(key)))) (quantize.py:235-241)
    on random configurations vs the oracle's Philox restatement."""
    from qsdp.quantize import quantize_bucket
    rng = np.random.default_rng(77)
    for t in range(30):
        bits = int(rng.integers(1, 17))
        inner = int(rng.integers(0, 2))
        n = int(rng.integers(1, 700))
        key = tuple(int(v) for v in rng.integers(0, 2**33, 5))
        start = int(rng.integers(0, 2**40))
        v = rng.standard_normal(n) * float(rng.choice([1e-3, 0.02, 3.0]))
        gen = np.random.Generator(np.random.Philox(np.random.SeedSequence(key + (start,))))
        blk = quantize_bucket(v, bits, "shift" if inner == 0 else "uniform_stochastic", gen)
        codes, meta, _ = oracle.quantize_segment(v, start, n, bits, inner, key, 1, noise=1)
        assert np.array_equal(oracle.unpack(codes, n, bits), blk.codes), t
        assert (float(meta[0, 0]), float(meta[0, 1]), float(meta[0, 2])) == (blk.shift, blk.scale_lo, blk.scale_hi), t


@pytest.mark.parametrize("P", [1, 2, 4])
def test_criterion7_oracle_hooks_100_steps(P):
    """Acceptance criterion 7 (test_acceptance.py:258-290) through the oracle-hooked
    workload: 100 steps bit-identical to the reference's ShardedMLP / ReferenceMLP golden run."""
    import mlp_workload as W
    from paper_2302_02390_b200.sharded import QuantConfig
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_mlp100.npz"))
    sim = W.make("oracle", widths=(64, 64, 10), P=P, batch=32, lr=0.05,
                 quant=QuantConfig(weight_bits=8, gradient_bits=8, bucket_size=1024), seed=11)
    losses, ag, rs = [], [], []
    for t in range(100):
        loss, e = sim.train_step(t)
        losses.append(loss)
        ag.append(e.allgather_bits)
        rs.append(e.reducescatter_bits)
    assert losses == list(g[f"P{P}_losses"])
    assert ag == list(g[f"P{P}_bits"][0]) and rs == list(g[f"P{P}_bits"][1])
    for name, v in sim.full_params().items():
        assert np.array_equal(v, g[f"P{P}_param_{name}"]), name


def test_shared_generator_golden(oracle):
    """bucketed_quantize with one Generator across buckets (quantize.py:289-313):
    codes, scales and where the stream is left, vs the reference goldens."""
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_shared.npz"))
    for i, (bits, inner, S, n, seed) in enumerate(g["sh_cases"]):
        bg = np.random.PCG64(int(seed))
        st = bg.state["state"]
        codes, meta, bad, (s2, inc2) = oracle.quantize_shared(g[f"sh_{i}_x"], int(S), int(bits), int(inner),
                                                              int(st["state"]), int(st["inc"]))
        assert bad == -1
        assert np.array_equal(codes, g[f"sh_{i}_codes"]) and np.array_equal(meta, g[f"sh_{i}_meta"]), i
        bg.state = {"bit_generator": "PCG64", "state": {"state": s2, "inc": inc2}, "has_uint32": 0, "uinteger": 0}
        assert int(bg.random_raw()) == int(g[f"sh_{i}_next"][0]), i
