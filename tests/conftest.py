import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REFERENCE_SRC = "/root/reference/pkg/src"
GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")
GOLDEN_PHILOX = os.path.join(ROOT, "tests", "golden", "golden_philox.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device and the built libqsdp_b200.so")
    config.addinivalue_line("markers", "reference: needs the live reference under /root/reference")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    has_ref = os.path.isdir(REFERENCE_SRC)
    skip_gpu = pytest.mark.skip(reason="no CUDA device")
    skip_ref = pytest.mark.skip(reason="/root/reference not mounted")
    for item in items:
        if "gpu" in item.keywords and not has_gpu:
            item.add_marker(skip_gpu)
        if "reference" in item.keywords and not has_ref:
            item.add_marker(skip_ref)


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN, allow_pickle=False)


@pytest.fixture(scope="session")
def golden_philox():
    return np.load(GOLDEN_PHILOX, allow_pickle=False)


def golden_philox_cases(g):
    """The quantizer cases of golden_philox.npz (reference quantize_bucket + numpy Philox)."""
    for i, r in enumerate(g["phq_cases"]):
        bits, inner, S, n, start, root, step, layer, phase, worker = (int(v) for v in r)
        yield dict(i=i, bits=bits, inner=inner, bucket=S, n=n, start=start, key=(root, step, layer, phase, worker),
                   x=g[f"phq_{i}_x"], codes=g[f"phq_{i}_codes"], meta=g[f"phq_{i}_meta"], deq=g[f"phq_{i}_deq"])


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.lib()
    return O


@pytest.fixture(scope="session")
def reference():
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    import qsdp  # noqa: F401
    return qsdp


def golden_cases(g):
    """Yield dicts describing each golden quantizer case."""
    rows = g["quant_cases"]
    for i, r in enumerate(rows):
        bits, inner, S, n, start, root, step, layer, phase, worker = (int(v) for v in r)
        yield dict(i=i, bits=bits, inner=inner, bucket=S, n=n, start=start,
                   key=(root, step, layer, phase, worker),
                   x=g[f"quant_{i}_x"], codes=g[f"quant_{i}_codes"], meta=g[f"quant_{i}_meta"],
                   deq=g[f"quant_{i}_deq"], wire=g[f"quant_{i}_wire"])


def golden_hooks(g):
    for h in range(int(g["n_hooks"])):
        run, kind, step, layer, phase = (int(v) for v in g[f"hookmeta_{h}"])
        P, wb, gb, S, seed = (int(v) for v in g[f"run_{run}_cfg"])
        yield dict(h=h, run=run, kind="ag" if kind == 0 else "rs", step=step, layer=layer, phase=phase,
                   P=P, wbits=wb, gbits=gb, bucket=S, seed=seed,
                   inp=g[f"hook_{h}_in"], out=g[f"hook_{h}_out"])


def golden_level_cases(g):
    """Yield the inner="levels" golden cases (quantize.py:225-286, 400-422)."""
    for k, (ti, bits, S, n) in enumerate(g["lv_cases"]):
        yield dict(k=k, table=g[f"lvtab_{int(ti)}"], bits=int(bits), bucket=int(S), n=int(n),
                   x=g[f"lv_{k}_x"], codes=g[f"lv_{k}_codes"], meta=g[f"lv_{k}_meta"], deq=g[f"lv_{k}_deq"])


def golden_learn_cases(g):
    """Yield the learn_levels golden cases (quantize.py:366-397)."""
    for k, lr in enumerate(g["ll_lr"]):
        yield dict(k=k, lr=float(lr), values=g[f"ll_{k}_values"], init=g[f"ll_{k}_init"], out=g[f"ll_{k}_out"])
