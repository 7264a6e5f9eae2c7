"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel."""
import collections
import csv
import sys


def main(path, frames):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == 'ID':
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    unit = ''
    for d in data:
        if d['Metric Name'] != 'gpu__time_duration.sum':
            continue
        unit = d['Metric Unit']
        name = d['Kernel Name'].split('(')[0].replace('void ', '').replace('(anonymous namespace)::', '')
        agg[name][0] += 1
        agg[name][1] += float(d['Metric Value'].replace(',', ''))
    scale = {'ns': 1e-3, 'usecond': 1.0, 'us': 1.0, 'msecond': 1e3, 'ms': 1e3}.get(unit, 1.0)
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':60s} {'launches/frame':>14s} {'us/frame':>10s} {'share':>7s}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:60]:60s} {v[0] / frames:14.1f} {v[1] * scale / frames:10.1f} {100 * v[1] / tot:6.1f}%")
    print(f"{'total':60s} {sum(v[0] for v in agg.values()) / frames:14.1f} {tot * scale / frames:10.1f}")


if __name__ == '__main__':
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1.0)
