"""Summarise an ncu launch list (gpu__time_duration per launch) by kernel: count, total, share."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    hdr = rows[h]
    ki, vi, ui = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Unit')
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[h + 1:]:
        v = float(r[vi].replace(',', ''))
        v *= {'nsecond': 1e-3, 'ns': 1e-3, 'usecond': 1.0, 'us': 1.0, 'msecond': 1e3, 'ms': 1e3}.get(r[ui], 1.0)
        name = r[ki]
        short = ('sweep_kernel<' + name.split('sweep_kernel<')[1].split('>')[0] + '>') if 'sweep_kernel<' in name \
            else name.split('(')[0].split('::')[-1][:60]
        agg[short][0] += 1
        agg[short][1] += v
    tot = sum(t for _, t in agg.values())
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:45s} n={c:5d} total={t / 1e3:9.2f} ms avg={t / c:8.1f} us share={100 * t / tot:5.1f}%")
    print(f"total {tot / 1e3:.2f} ms")


if __name__ == "__main__":
    main(sys.argv[1])
