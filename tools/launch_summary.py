"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel.

python tools/launch_summary.py <launches.csv> [header line ...]
"""
import collections
import csv
import sys


def main(path, header):
    rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[12] == "gpu__time_duration.sum"]
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        name = r[4].split("(")[0][:60]
        tot[name] += float(r[14]) / 1e3
        cnt[name] += 1
    all_us = sum(tot.values())
    for h in header:
        print(h)
    for name, us in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{name:62s} n={cnt[name]:3d} total={us:11.1f} us  share={100 * us / all_us:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
