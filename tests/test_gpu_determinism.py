"""GPU: run-twice bitwise determinism (SURVEY §5's race check, in place of compute-sanitizer,
which this pool does not allow).  The same collectives -- fused all-gathers and
reduce-scatters over several communicators -- run once serially on one stream and then
repeatedly with every communicator on its own stream, all in flight together (the bench's
schedule, grids capped to share SMs); every output must be bit-identical each time.  A race
in the persistent quantizer's shared-memory ring, the per-warp seed / dequant tables or the
slot writes would show up as a difference."""

import numpy as np
import pytest
import torch

from paper_2302_02390_b200.comm import QSDPComm
from paper_2302_02390_b200.quantize import QuantSpec, SegmentKey

pytestmark = pytest.mark.gpu


def _run(comms, xs, gs, outs, shards, streams, ctas):
    cur = torch.cuda.current_stream()
    for i, c in enumerate(comms):
        s = streams[i] if streams else cur
        c.set_ctas_per_sm(ctas)
        if streams:
            s.wait_stream(cur)
        with torch.cuda.stream(s):
            n = xs[i].numel()
            c.all_gather(xs[i], [(0, n)], SegmentKey(7, 3, i, 0, 0), outs[i])
            c.reduce_scatter(gs[i], [(0, n)], SegmentKey(7, 3, i, 2, 0), shards[i])
    if streams:
        for s in streams:
            cur.wait_stream(s)
    torch.cuda.synchronize()
    return [o.clone() for o in outs] + [s.clone() for s in shards]


@pytest.mark.parametrize("gbits", [8, 4])
def test_concurrent_collectives_bitwise_deterministic(gbits):
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev).manual_seed(11)
    sizes = [7_077_888, 1_000_003, 3 * 1024 * 1024, 65_536 + 17, 38_633_472 // 4]
    comms = [QSDPComm(n, QuantSpec(8, 1024, "shift"), QuantSpec(gbits, 1024, "uniform_stochastic"), device=dev)
             for n in sizes]
    xs = [torch.randn(n, generator=gen, device=dev) * 0.02 for n in sizes]
    gs = [torch.randn(n, generator=gen, device=dev) * 1e-3 for n in sizes]
    outs = [torch.empty(n, device=dev) for n in sizes]
    shards = [torch.empty(n, device=dev) for n in sizes]
    ref = _run(comms, xs, gs, outs, shards, None, 0)
    streams = [torch.cuda.Stream(device=dev) for _ in sizes]
    for rep, ctas in enumerate((0, 1, 1)):
        for o in outs + shards:
            o.fill_(float("nan"))
        got = _run(comms, xs, gs, outs, shards, streams, ctas)
        for k, (a, b) in enumerate(zip(ref, got)):
            assert torch.equal(a.view(torch.int32), b.view(torch.int32)), (rep, k)
    for c in comms:
        c.close()
    assert all(np.isfinite(r.cpu().numpy()).all() for r in ref)
