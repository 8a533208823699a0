"""Per-kernel durations from an ncu launch list CSV (the
`--metrics gpu__time_duration.sum --clock-control none --csv` pass):
mean per kernel name, launches and share of the total.

usage: python scripts/launch_summary.py launches.csv [filter-substring ...]
"""
import csv
import sys
from collections import defaultdict


def main():
    path, filt = sys.argv[1], sys.argv[2:]
    rows = list(csv.reader(open(path)))
    head = None
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if "Kernel Name" in r:
            head = r
            continue
        if head and len(r) == len(head):
            d = dict(zip(head, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            n = d["Kernel Name"]
            tot[n] += float(d["Metric Value"]) / 1e6
            cnt[n] += 1
    total = sum(tot.values())
    for n, t in sorted(tot.items(), key=lambda kv: -kv[1]):
        if filt and not any(f in n for f in filt):
            continue
        print(f"{n[:70]:70s} launches={cnt[n]:3d} mean={t / cnt[n]:9.4f} ms total={t:9.3f} ms share={100 * t / total:6.2f}%")


if __name__ == "__main__":
    main()
