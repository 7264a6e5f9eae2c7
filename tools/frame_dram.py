"""Summarise tools/frame_metrics.sh's launch list: per kernel of one frame (the last
of the run) duration, DRAM bytes and fp64 instruction counts; the frame's measured DRAM
total. Usage: python tools/frame_dram.py gpurun_out/TAG_frame.csv [out.json]"""
import collections
import csv
import json
import re
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, launches = None, collections.OrderedDict()
    for r in rows:
        if r and r[0] == 'ID':
            hdr = r
            continue
        if not (hdr and len(r) == len(hdr)):
            continue
        d = dict(zip(hdr, r))
        L = launches.setdefault(d['ID'], {'name': d['Kernel Name']})
        try:
            v = float(d['Metric Value'].replace(',', ''))
        except ValueError:
            continue
        u = d['Metric Unit']
        if d['Metric Name'].startswith('dram__bytes'):
            v *= {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}.get(u, 1)
        if d['Metric Name'] == 'gpu__time_duration.sum':
            v *= {'ns': 1, 'usecond': 1e3, 'msecond': 1e6}.get(u, 1)
        L[d['Metric Name']] = v
    return list(launches.values())


def main(path, out=None):
    ls = load(path)
    starts = [i for i, l in enumerate(ls) if 'preprocess_kernel' in l['name']]
    frame = ls[starts[-1]:]
    agg = collections.OrderedDict()
    for l in frame:
        n = re.sub(r'\(.*', '', l['name'].replace('(anonymous namespace)::', '').replace('void ', ''))
        a = agg.setdefault(n, collections.Counter())
        a['launches'] += 1
        for k, v in l.items():
            if k != 'name' and not k.endswith('pct'):
                a[k] += v
    tot = collections.Counter()
    print(f"{'kernel':40s} {'n':>3s} {'us':>9s} {'DRAM MB':>9s} {'GB/s':>8s} {'DFMA M':>8s}")
    for n, a in agg.items():
        mb = (a['dram__bytes_read.sum'] + a['dram__bytes_write.sum']) / 1e6
        us = a['gpu__time_duration.sum'] / 1e3
        print(f"{n[:40]:40s} {a['launches']:3d} {us:9.1f} {mb:9.1f} {mb / 1e3 / (us / 1e6) if us else 0:8.1f} "
              f"{a['sm__sass_thread_inst_executed_op_dfma_pred_on.sum'] / 1e6:8.1f}")
        tot.update(a)
    mb = (tot['dram__bytes_read.sum'] + tot['dram__bytes_write.sum']) / 1e6
    print(f"frame total: {tot['gpu__time_duration.sum'] / 1e3:.1f} us serialized, DRAM {mb:.1f} MB")
    if out:
        comp = next(v for k, v in agg.items() if 'composite_kernel' in k)
        json.dump({"frame_dram_bytes": tot['dram__bytes_read.sum'] + tot['dram__bytes_write.sum'],
                   "frame_kernel_us_serialized": tot['gpu__time_duration.sum'] / 1e3,
                   "composite": {"dfma": comp['sm__sass_thread_inst_executed_op_dfma_pred_on.sum'],
                                 "dmul": comp['sm__sass_thread_inst_executed_op_dmul_pred_on.sum'],
                                 "dadd": comp['sm__sass_thread_inst_executed_op_dadd_pred_on.sum'],
                                 "dram_bytes": comp['dram__bytes_read.sum'] + comp['dram__bytes_write.sum'],
                                 "us": comp['gpu__time_duration.sum'] / 1e3},
                   "kernels": {k: {"launches": v['launches'], "us": v['gpu__time_duration.sum'] / 1e3,
                                   "dram_bytes": v['dram__bytes_read.sum'] + v['dram__bytes_write.sum']}
                               for k, v in agg.items()},
                   "source": path}, open(out, 'w'), indent=1)


if __name__ == '__main__':
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
