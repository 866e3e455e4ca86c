"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel:
launches, total/avg device time and share.  usage: launch_summary.py launches.csv"""
import collections
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
    h = rows[hi]
    ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        scale = {'ns': 1e-3, 'us': 1.0, 'usecond': 1.0, 'nsecond': 1e-3, 'ms': 1e3}.get(r[ui], 1e-3)
        a = agg.setdefault(r[ki].split('(')[0][:70], [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(',', '')) * scale
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':70s} {'launches':>8s} {'total_us':>10s} {'share':>6s} {'avg_us':>8s}")
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:70s} {a[0]:8d} {a[1]:10.1f} {100 * a[1] / tot:5.1f}% {a[1] / a[0]:8.2f}")


if __name__ == '__main__':
    main()
