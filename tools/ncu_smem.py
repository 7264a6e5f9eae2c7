"""Source lines of an ncu report ranked by shared-memory wavefronts (ideal vs actual:
the excess is bank conflicts).  Usage: python tools/ncu_smem.py report.ncu-rep [top]"""
import csv
import subprocess
import sys


def main(path, top=25):
    out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, fname, lines = None, '', []
    for r in rows:
        if r and r[0] in ('File Name', 'File Path'):
            fname = r[1].split('/')[-1]
        if r and r[0] == 'Line No':
            hdr = r
            continue
        if hdr and r and r[0].isdigit():
            d = dict(zip(hdr, r))
            try:
                w = float(d.get('L1 Wavefronts Shared', '0') or 0)
                wi = float(d.get('L1 Wavefronts Shared Ideal', '0') or 0)
                inst = float(d.get('Instructions Executed', '0') or 0)
            except ValueError:
                continue
            if w:
                lines.append((w, wi, inst, f"{fname}:{r[0]}", r[1].strip()[:70]))
    tot = sum(x[0] for x in lines) or 1
    print(f"total shared wavefronts {tot:.3e}, ideal {sum(x[1] for x in lines):.3e}")
    for w, wi, inst, loc, src in sorted(lines, reverse=True)[:top]:
        print(f"{100 * w / tot:5.1f}% {loc:26s} wf={w:10.3e} ideal={wi:10.3e} inst={inst:10.3e} {src}")


if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
