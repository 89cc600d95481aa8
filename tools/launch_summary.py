"""Summarise an ncu --metrics gpu__time_duration.sum launch list (second half = measured build)."""
import collections
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    data = rows[hi + 1:]
    ki, vi, ii = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
    half = data[len(data) // 2:] if len(sys.argv) < 3 else data
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in half:
        v = float(r[vi].replace(",", ""))
        agg[r[ki][:90]][0] += 1
        agg[r[ki][:90]][1] += v
        tot += v
    print(f"launches={len(half)} total={tot / 1e6:.3f} ms")
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
        print(f"{v / 1e6:8.3f} ms {100 * v / tot:5.1f}% n={c:4d} {k}")


if __name__ == "__main__":
    main()
