"""Per-kernel summary of an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python scripts/launch_summary.py launches.csv "<command that produced it>" > summary.txt
'share' is over every launch of the command; 'hot share' is over the K1-K4 hot-path kernels, to set
against the bench line's kernels.*.share_of_step (ncu times are cold-cache and serialised)."""
import collections
import csv
import sys

HOT = {"K1 quantize (shift)", "K2 quantize (stochastic)", "K3 dequantize", "K4 dequant-accumulate"}


def label(name: str) -> str:
    if "quantize_tma32_kernel" in name or "quantize_tma_kernel" in name or "quantize_kernel" in name:
        inner = name.split("<")[1].split(",")[1].strip()
        return "K1 quantize (shift)" if inner in ("0", "(int)0") else "K2 quantize (stochastic)"
    if "dequant_kernel" in name or "dequant_fast" in name:
        parts = [p.strip() for p in name.split("<")[1].split(">")[0].split(",")]
        acc = parts[4] if len(parts) > 4 else "0"
        return "K4 dequant-accumulate" if acc in ("1", "true", "(bool)1") else "K3 dequantize"
    base = name.split("(")[0].replace("void ", "")
    base = base.split("<")[0]
    return base.replace("qsdp::", "")


def main():
    path, cmd = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(lines))
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        v = v * 1e-3 if r["Metric Unit"] == "ns" else v if r["Metric Unit"] == "us" else v * 1e3
        k = label(r["Kernel Name"])
        tot[k] += v
        cnt[k] += 1
    allt = sum(tot.values())
    hot = sum(t for k, t in tot.items() if k in HOT)
    print(f"# {cmd}")
    print("# per-launch times are cold-cache and serialised (ncu).  'share' is over every launch of the command;")
    print("# 'hot share' is over K1-K4, to set against the bench line's kernels.*.share_of_step.")
    print(f"{'kernel':40s} {'launches':>8s} {'total ms':>10s} {'share':>7s} {'hot share':>9s} {'avg us':>9s}")
    for k, t in sorted(tot.items(), key=lambda kv: -kv[1]):
        hs = f"{t / hot:9.3f}" if k in HOT and hot else " " * 9
        print(f"{k[:40]:40s} {cnt[k]:8d} {t / 1e3:10.3f} {t / allt:7.3f} {hs} {t / cnt[k]:9.2f}")


if __name__ == "__main__":
    main()
