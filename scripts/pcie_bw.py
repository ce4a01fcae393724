"""Raw pinned-host <-> HBM copy bandwidth (the ceiling of bench.py's e2e number).

    python scripts/pcie_bw.py
Times 1 GB H2D alone, 0.5 GB D2H alone, and both concurrently on two streams (CUDA events)."""
import json

import torch

dev = torch.device("cuda", 0)
hb = torch.empty(1 << 28, dtype=torch.float32).pin_memory()  # 1 GiB
ho = torch.empty(1 << 27, dtype=torch.float32).pin_memory()
db = torch.empty(1 << 28, dtype=torch.float32, device=dev)
do = torch.randn(1 << 27, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        main = torch.cuda.current_stream()
        for s in (s1, s2):
            s.wait_stream(main)
        if h2d:
            with torch.cuda.stream(s1):
                db.copy_(hb, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                ho.copy_(do, non_blocking=True)
        main.wait_stream(s1)
        main.wait_stream(s2)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1e-3)
    return best


t1 = run(True, False)
t2 = run(False, True)
t3 = run(True, True)
print(json.dumps({"h2d_gbs": round(hb.numel() * 4 / t1 / 1e9, 1), "d2h_gbs": round(ho.numel() * 4 / t2 / 1e9, 1),
                  "both_ms": round(t3 * 1e3, 2), "both_h2d_equiv_gbs": round(hb.numel() * 4 / t3 / 1e9, 1)}))
