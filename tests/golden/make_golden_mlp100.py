"""Golden runs of the reference's acceptance criterion 7 (pkg/tests/test_acceptance.py:258-290):
ShardedMLP and ReferenceMLP, widths (64, 64, 10), batch 32, lr 0.05, w8/g8 bucket 1024, seeds 11,
100 training steps, P in {1, 2, 4} (dev container only: the reference does not travel):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_mlp100.py

Writes tests/golden/golden_mlp100.npz: per P the 100 losses, the per-step ledger bits
(allgather, reducescatter) and the final full parameters (ShardedMLP == ReferenceMLP,
asserted here as the reference's criterion 7 does)."""

from __future__ import annotations

import os

import numpy as np
from qsdp.sharded import QuantConfig, ReferenceMLP, ShardedMLP, SimConfig

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_mlp100.npz")


def main():
    out = {"numpy_version": np.array(np.__version__), "steps": np.array(100)}
    for P in (1, 2, 4):
        cfg = SimConfig(widths=(64, 64, 10), P=P, batch=32, lr=0.05,
                        quant=QuantConfig(weight_bits=8, gradient_bits=8, bucket_size=1024),
                        root_seed=11, param_seed=11, data_seed=11)
        sim, ref = ShardedMLP(cfg), ReferenceMLP(cfg)
        losses, ag, rs = [], [], []
        for t in range(100):
            loss, entry = sim.train_step(t)
            ref.train_step(t)
            losses.append(loss)
            ag.append(entry.allgather_bits)
            rs.append(entry.reducescatter_bits)
        for name, full in sim.full_params().items():
            assert np.array_equal(full, ref.params[name]), (P, name)  # criterion 7
            out[f"P{P}_param_{name}"] = full
        out[f"P{P}_losses"] = np.array(losses)
        out[f"P{P}_bits"] = np.array([ag, rs], dtype=np.int64)
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT} ({os.path.getsize(OUT) / 1e3:.1f} kB)")


if __name__ == "__main__":
    main()
