"""Sum instructions and stall samples of an ncu source page over named line ranges.
Usage: python tools/ncu_phases.py report.ncu-rep file.cu "name:lo-hi" ... (other files -> 'helpers')"""
import csv
import subprocess
import sys


def main(path, fname, ranges):
    out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, cur = None, ''
    agg = {}
    for r in rows:
        if r and r[0] == 'File Path':
            cur = r[1].split('/')[-1]
        if r and r[0] == 'Line No':
            hdr = r
            continue
        if not (hdr and r and r[0].isdigit()):
            continue
        d = dict(zip(hdr[4:], r[4:]))
        try:
            inst = int(d.get('Instructions Executed', '0') or 0)
            smp = int(d.get('Warp Stall Sampling (All Samples)', '0') or 0)
        except ValueError:
            continue
        ln = int(r[0])
        name = cur if cur != fname else 'other'
        if cur == fname:
            for nm, lo, hi in ranges:
                if lo <= ln <= hi:
                    name = nm
                    break
        a = agg.setdefault(name, [0, 0])
        a[0] += inst
        a[1] += smp
    ti = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    for k, (i, s) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:24s} inst {i / 1e6:8.1f}M ({100 * i / ti:5.1f}%)  samples {100 * s / ts:5.1f}%")


if __name__ == '__main__':
    rs = []
    for a in sys.argv[3:]:
        nm, span = a.split(':')
        lo, hi = span.split('-')
        rs.append((nm, int(lo), int(hi)))
    main(sys.argv[1], sys.argv[2], rs)
