"""Summarize an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections
import csv
import sys


def main(path, title=""):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Unit')
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        if len(r) <= vi:
            continue
        name = r[ki].split('(')[0].replace('void ', '').replace('fnlh::<unnamed>::', '').replace('unnamed>::', '')
        v = float(r[vi].replace(',', '')) * {'nsecond': 1, 'usecond': 1e3, 'msecond': 1e6}.get(r[ui], 1)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"# {title}")
    print(f"# launches {sum(v[0] for v in agg.values())}  total {tot / 1e6:.3f} ms (cold-cache, serialized: compare SHARES)")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:50s} {v[0]:6d} {v[1] / 1e6:9.3f} ms {100 * v[1] / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
