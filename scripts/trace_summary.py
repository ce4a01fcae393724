"""Summarise a torch.profiler chrome trace: GPU span, busy time (union of kernel intervals),
kernel time by category and by stream, top kernels.  python scripts/trace_summary.py T.json"""
import collections
import json
import sys


def cat(name):
    n = name.lower()
    if "qsdp" in n:
        return "qsdp"
    if "nccl" in n:
        return "nccl"
    if "gemm" in n or "cutlass" in n or "sm90" in n or "sm100" in n or "nvjet" in n or "cublas" in n:
        return "gemm"
    if "flash" in n or "fmha" in n or "attention" in n or "sdpa" in n:
        return "attention"
    if "adam" in n or "multi_tensor" in n:
        return "optimizer"
    if "memcpy" in n or "memset" in n:
        return "copy"
    return "elementwise/other"


def main(path):
    ev = json.load(open(path))["traceEvents"]
    ks = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
    if not ks:
        print("no kernels")
        return
    t0 = min(e["ts"] for e in ks)
    t1 = max(e["ts"] + e["dur"] for e in ks)
    iv = sorted((e["ts"], e["ts"] + e["dur"]) for e in ks)
    busy, cs, ce = 0.0, None, None
    for s, e in iv:
        if ce is None or s > ce:
            if ce is not None:
                busy += ce - cs
            cs, ce = s, e
        else:
            ce = max(ce, e)
    busy += ce - cs
    bycat, bystream, byname = (collections.defaultdict(float) for _ in range(3))
    cnt = collections.Counter()
    for e in ks:
        bycat[cat(e["name"])] += e["dur"]
        bystream[e.get("tid")] += e["dur"]
        k = e["name"][:90]
        byname[k] += e["dur"]
        cnt[k] += 1
    print(f"span {1e-3 * (t1 - t0):.2f} ms  busy(union) {1e-3 * busy:.2f} ms  kernels {len(ks)}  "
          f"sum {1e-3 * sum(e['dur'] for e in ks):.2f} ms")
    print("by category (ms):", {k: round(v * 1e-3, 2) for k, v in sorted(bycat.items(), key=lambda x: -x[1])})
    print("by stream (ms):", {k: round(v * 1e-3, 2) for k, v in sorted(bystream.items(), key=lambda x: -x[1])})
    for k, v in sorted(byname.items(), key=lambda x: -x[1])[:15]:
        print(f"  {v * 1e-3:8.2f} ms  x{cnt[k]:5d}  {k}")
    # host side: CUDA runtime calls by name, and the launches of each kernel category
    corr = {e.get("args", {}).get("correlation"): cat(e["name"]) for e in ks}
    rt = collections.defaultdict(float)
    rtc = collections.Counter()
    lc = collections.defaultdict(float)
    lcc = collections.Counter()
    for e in ev:
        if e.get("ph") == "X" and e.get("cat") == "cuda_runtime":
            rt[e["name"]] += e["dur"]
            rtc[e["name"]] += 1
            c = corr.get(e.get("args", {}).get("correlation"))
            if c is not None and "aunch" in e["name"]:
                lc[c] += e["dur"]
                lcc[c] += 1
    if rt:
        print("CUDA runtime (ms, count):", {k: (round(v * 1e-3, 2), rtc[k]) for k, v in
                                             sorted(rt.items(), key=lambda x: -x[1])[:8]})
        print("launch time by kernel category (ms, count, us/launch):",
              {k: (round(v * 1e-3, 2), lcc[k], round(v / max(lcc[k], 1), 1)) for k, v in lc.items()})
    # host side: user annotations (FSDP2's record_function ranges, optimizer, ...) by name
    ann = collections.defaultdict(float)
    acnt = collections.Counter()
    for e in ev:
        if e.get("ph") == "X" and e.get("cat") == "user_annotation":
            ann[e["name"][:70]] += e["dur"]
            acnt[e["name"][:70]] += 1
    if ann:
        print("host annotations (ms, count):")
        for k, v in sorted(ann.items(), key=lambda x: -x[1])[:20]:
            print(f"  {v * 1e-3:8.2f} ms  x{acnt[k]:5d}  {k}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("==", p)
        main(p)
