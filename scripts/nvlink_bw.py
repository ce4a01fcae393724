"""NVLink write bandwidth on this box, by store method (one process, all visible GPUs):
per-lane 16-byte stores, TMA bulk stores (4 KB chunks, 2 or 4 in flight per warp), and the
copy engines (tensor.copy_ to a peer).  Scenarios: GPU 0 -> one peer, GPU 0 -> every peer
(the push all-gather's fan-out), every GPU -> every peer at once.  GB/s = bytes leaving
each GPU / time (per direction; 900 GB/s is the NVLink 5 figure).

    make -C scripts/nvlbw && python scripts/nvlink_bw.py [MB]"""
import ctypes
import json
import os
import sys

import torch

here = os.path.dirname(os.path.abspath(__file__))
L = ctypes.CDLL(os.path.join(here, "nvlbw", "libnvlbw.so"))
L.nvlbw_run.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p), ctypes.c_int,
                        ctypes.c_longlong, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
n = torch.cuda.device_count()
assert L.nvlbw_enable_peers(n) == 0
mb = int(sys.argv[1]) if len(sys.argv) > 1 else 256
nbytes = mb << 20
src = [torch.randint(0, 255, (nbytes,), dtype=torch.uint8, device=f"cuda:{i}") for i in range(n)]
# dst[i][j]: buffer on GPU j receiving from GPU i
dst = [[torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{j}") if j != i else None for j in range(n)]
       for i in range(n)]
streams = [torch.cuda.Stream(device=i) for i in range(n)]


def launch(i, peers, mode):
    with torch.cuda.device(i):
        s = streams[i]
        if mode == "ce":
            for j in peers:
                with torch.cuda.stream(s):
                    dst[i][j].copy_(src[i], non_blocking=True)
            return
        arr = (ctypes.c_void_p * len(peers))(*[dst[i][j].data_ptr() for j in peers])
        m = {"st16": 0, "tma2": 2, "tma4": 4}[mode]
        grid = 148 * (4 if m == 0 else 2)
        rc = L.nvlbw_run(m, src[i].data_ptr(), arr, len(peers), nbytes, grid, 256, s.cuda_stream)
        assert rc == 0, rc


def run(senders, fan, mode, reps=5):
    peers = {i: ([j for j in range(n) if j != i][:fan]) for i in senders}
    for _ in range(2):
        for i in senders:
            launch(i, peers[i], mode)
    for i in range(n):
        torch.cuda.synchronize(i)
    ev = {i: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for i in senders}
    for i in senders:
        ev[i][0].record(streams[i])
    for _ in range(reps):
        for i in senders:
            launch(i, peers[i], mode)
    for i in senders:
        ev[i][1].record(streams[i])
    for i in range(n):
        torch.cuda.synchronize(i)
    t = max(ev[i][0].elapsed_time(ev[i][1]) for i in senders) / reps * 1e-3
    return round(nbytes * fan / t / 1e9, 1)


res = {"gpus": n, "mb": mb}
if n >= 2:
    for mode in ("st16", "tma2", "tma4", "ce"):
        res[f"{mode}_0to1"] = run([0], 1, mode)
        res[f"{mode}_0toall"] = run([0], n - 1, mode)
        res[f"{mode}_alltoall"] = run(list(range(n)), n - 1, mode)
print(json.dumps(res), flush=True)
