"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list.

usage: python tools/launch_summary.py gpurun_out/launches_TAG.csv [> profiles/…]
Per kernel: launches, total/avg device time and share (cold-cache, serialised
launches: compare SHARES with bench.py, not absolutes)."""
import collections
import csv
import re
import sys


def short(name):
    name = name.replace("(anonymous namespace)::", "")
    m = re.search(r"([A-Za-z_][\w:]*(?:<[^()]*?>)?)\(", name)
    s = m.group(1) if m else name
    return s.replace("dass::", "")


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    for r in rows[hi + 1:]:
        if len(r) <= vi or not r[vi]:
            continue
        k = short(r[ki])
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':58s} {'n':>6s} {'total ms':>10s} {'avg us':>10s} {'share':>7s}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:58]:58s} {v[0]:6d} {v[1] / 1e3:10.3f} {v[1] / v[0]:10.2f} {v[1] / tot * 100:6.1f}%")
    print(f"{'TOTAL':58s} {sum(v[0] for v in agg.values()):6d} {tot / 1e3:10.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
