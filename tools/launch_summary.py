"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel count, total, share."""
import collections
import csv
import sys


def summarise(path):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for x in csv.DictReader(lines):
        if x["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(x["Metric Value"].replace(",", ""))
        v *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(x["Metric Unit"], 1e-6)
        k = x["Kernel Name"].split("(")[0][:70]
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v[1] for v in agg.values())
    out = [f"{'launches':>8} {'total_ms':>11} {'share':>6} {'avg_us':>10}  kernel"]
    for k, (c, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"{c:8d} {ms:11.3f} {100 * ms / tot:5.1f}% {1e3 * ms / c:10.1f}  {k}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
