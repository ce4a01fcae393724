"""GPU: QSDP comms inside FSDP2 -- a short GPT run tracks the unquantized run."""

import os
import subprocess
import sys

import pytest
import torch

from conftest import ROOT

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("ngpu", [2, 4])
def test_fsdp2_qsdp_tracks_fsdp(ngpu):
    """World >= 2 only: at world 1 FSDP2 runs no collective, so QSDP would never be exercised."""
    if torch.cuda.device_count() < ngpu:
        pytest.skip(f"needs {ngpu} GPUs")
    env = dict(os.environ, PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={ngpu}",
                        "--master-addr", "127.0.0.1", "--master-port", str(29600 + ngpu),
                        os.path.join(ROOT, "tests", "dist_fsdp_check.py")],
                       capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
