"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import csv
import sys
from collections import defaultdict


def main(path, top=30, by_name=False):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    gi = h.index("Grid Size")
    agg = defaultdict(lambda: [0, 0.0])
    tot = 0.0
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
    for r in rows[hi + 1:]:
        v = float(r[vi].replace(",", "")) * scale[r[ui]]
        name = r[ki].split("(")[0].replace("gicp::<unnamed>::", "")[:60] + ("" if by_name else " " + r[gi])
        agg[name][0] += 1
        agg[name][1] += v
        tot += v
    print(f"{'us':>10s} {'share':>6s} {'n':>4s}  kernel grid")
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{v:10.1f} {100 * v / tot:5.1f}% {c:4d}  {k}")
    print(f"total {tot:.1f} us over {len(rows) - hi - 1} launches")


if __name__ == "__main__":
    main(sys.argv[1], by_name="--by-name" in sys.argv[2:])
