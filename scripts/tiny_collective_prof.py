import collections, os, sys, torch
sys.path.insert(0, "/root/repo")
from paper_2302_02390_b200.comm import QSDPComm, plan_segments
from paper_2302_02390_b200.quantize import QuantSpec, SegmentKey
dev = torch.device("cuda", 0)
comm = QSDPComm(1 << 20, QuantSpec(8, 1024, "shift"), QuantSpec(8, 1024, "uniform_stochastic"), device=dev)
tin, tout = torch.randn(1024, device=dev), torch.empty(1024, device=dev)
big, bout = torch.randn(1 << 20, device=dev), torch.empty(1 << 20, device=dev)
def run(x, o, k):
    for gi in range(k): comm.all_gather(x, [(0, x.numel())], SegmentKey(0, 0, gi, 0, 0), o)
for _ in range(3): run(tin, tout, 13)
torch.cuda.synchronize()
for name, x, o in (("tiny", tin, tout), ("1M", big, bout)):
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        run(x, o, 13); torch.cuda.synchronize()
    tot = collections.defaultdict(float); cnt = collections.Counter()
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            n = e.name.split("<")[0].split("(")[0].replace("void ", "").replace("qsdp::", "")
            tot[n] += e.device_time_total; cnt[n] += 1
    print(name, {k: (round(v / cnt[k], 2), cnt[k]) for k, v in tot.items()})
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g): run(x, o, 13)
    g.replay(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); 
    for _ in range(20): g.replay()
    b.record(); torch.cuda.synchronize()
    print(name, "graph per collective us:", round(a.elapsed_time(b) / 20 / 13 * 1e3, 2))
