"""Top source lines of an ncu report by warp-stall samples (needs -lineinfo and
--import-source on).  Usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import subprocess
import sys


def main(path, top=25):
    out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = None
    lines = []
    fname = ''
    for r in rows:
        if r and r[0] == 'File Path':
            fname = r[1].split('/')[-1]
        if r and r[0] == 'Line No':
            hdr = r
            continue
        if hdr and r and r[0] not in ('', '-'):
            d = dict(zip(hdr[4:], r[4:]))
            try:
                s = int(d.get('Warp Stall Sampling (All Samples)', '0'))
            except ValueError:
                continue
            stalls = {k: int(v) for k, v in d.items() if k.startswith('stall_') and '(' not in k and v.isdigit()}
            lines.append((s, f"{fname}:{r[0]}", r[1].strip()[:70], d.get('Instructions Executed', ''), stalls))
    tot = sum(x[0] for x in lines) or 1
    for s, loc, src, inst, st in sorted(lines, reverse=True)[:top]:
        topst = ', '.join(f"{k[6:]} {v}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3] if v)
        print(f"{100 * s / tot:5.1f}% {loc:22s} inst={inst:>10s} {src:70s} [{topst}]")


if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
