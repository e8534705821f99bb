"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) as markdown."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        if len(r) <= mi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")[:90]
        v = float(r[mi].replace(",", "")) * scale.get(r[ui], 1.0)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(t for _, t in agg.values())
    print(f"launches: {sum(n for n, _ in agg.values())}, total device time {tot:.2f} ms (cold-cache, serialised)\n")
    print("| kernel | launches | total ms | mean ms | share |")
    print("|---|---:|---:|---:|---:|")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k}` | {n} | {t:.3f} | {t / n:.4f} | {100 * t / tot:.1f}% |")


if __name__ == "__main__":
    main(sys.argv[1])
