"""Aggregate an ncu --metrics gpu__time_duration.sum CSV launch list per kernel."""
import csv, sys
from collections import defaultdict
def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]; ki = h.index("Kernel Name"); vi = h.index("Metric Value"); ui = h.index("Metric Unit")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    agg = defaultdict(lambda: [0, 0.0])
    scale = {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "second": 1e9, "s": 1e9}
    for r in rows[hi + 1:]:
        if len(r) <= vi or (mi is not None and r[mi] != "gpu__time_duration.sum"):
            continue
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        name = r[ki].split("(")[0][:80]
        agg[name][0] += 1; agg[name][1] += v
    tot = sum(v for _, v in agg.values())
    print(f"{'ms':>10} {'launches':>8} {'share':>6}  kernel")
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{v/1e6:10.3f} {c:8d} {100*v/tot:5.1f}%  {k}")
    print(f"{tot/1e6:10.3f} total ms (cold-cache, serialised)")
if __name__ == "__main__":
    main(sys.argv[1])
