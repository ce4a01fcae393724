"""The drop-in boundary against the unmodified reference class.

CPU half (this container, reference mounted): ``class B200ShardedMLP(QSDPHooks, ShardedMLP)``
composes with the live ``qsdp.sharded.ShardedMLP`` (sharded.py:308-503), the hooks replace
exactly the reference's two collective methods with the same parameters, every other method
(forward_layer / backward_layer / train_step) stays the reference's, and without a GPU the
composed object fails loudly instead of falling back to a CPU path.  The GPU half (the hooks'
results) is test_gpu_protocol.py: 100 criterion-7 steps bit-identical to the reference's
golden run.
"""

import inspect

import numpy as np
import pytest
import torch


@pytest.mark.reference
def test_hooks_override_exactly_the_reference_collectives(reference):
    from qsdp.sharded import ShardedMLP

    from paper_2302_02390_b200.sharded import QSDPHooks

    class B200ShardedMLP(QSDPHooks, ShardedMLP):
        pass

    for name in ("_gather", "_reduce_scatter"):
        assert getattr(B200ShardedMLP, name) is getattr(QSDPHooks, name)
        ref_params = list(inspect.signature(getattr(ShardedMLP, name)).parameters)
        ours = list(inspect.signature(getattr(QSDPHooks, name)).parameters)
        assert ours == ref_params, (name, ours, ref_params)
    for name in ("forward_layer", "backward_layer", "train_step", "run", "full_params", "__init__"):
        assert getattr(B200ShardedMLP, name) is getattr(ShardedMLP, name), name
    # the hooks touch only attributes the reference object has
    hooked = {"_gather", "_reduce_scatter"}
    own = {n for n, v in vars(QSDPHooks).items() if callable(v) and not n.startswith("__")}
    assert own - hooked <= {"_qsdp_dev", "_qsdp_quant"}


@pytest.mark.reference
def test_hook_records_are_reference_ledger_compatible(reference):
    """The hooks record their own Transfer rows into the reference's LedgerEntry: the fields
    LedgerEntry.record reads (sharded.py:148-157) exist with the reference's meaning."""
    from qsdp.sharded import LedgerEntry, Transfer as RT

    from paper_2302_02390_b200.sharded import Transfer

    a, b = LedgerEntry(step=0), LedgerEntry(step=0)
    for args in (("allgather", "d0", 8, 1040, 3, 8192), ("reducescatter", "d0", 8, 1040, 1, 8192),
                 ("allgather", "b0", 32, 40, 3, 320)):
        a.record(Transfer(*args))
        b.record(RT(*args))
    for f in ("allgather_bits", "reducescatter_bits", "allgather_payload_bits", "reducescatter_payload_bits"):
        assert getattr(a, f) == getattr(b, f), f
    assert [t.total_bits for t in a.transfers] == [t.total_bits for t in b.transfers]


@pytest.mark.reference
@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_composed_reference_fails_loudly_without_gpu(reference):
    from qsdp.sharded import QuantConfig, ShardedMLP, SimConfig

    from paper_2302_02390_b200.sharded import QSDPHooks

    class B200ShardedMLP(QSDPHooks, ShardedMLP):
        pass

    sim = B200ShardedMLP(SimConfig(widths=(64, 64, 10), P=4, batch=32, lr=0.05, quant=QuantConfig()))
    before = {k: np.copy(v) for k, v in sim.full_params().items()}
    with pytest.raises(RuntimeError, match="CUDA device"):
        sim.train_step(0)
    for k, v in sim.full_params().items():  # nothing was updated on a silent fallback
        assert np.array_equal(v, before[k])
