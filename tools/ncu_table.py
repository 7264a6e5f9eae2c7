"""Per-launch table of an ncu report (--set full): duration, DRAM bytes and GB/s,
L2 / L1 hit rates, achieved occupancy, issue-slot use.  Usage:
python tools/ncu_table.py report.ncu-rep"""
import csv
import re
import subprocess
import sys

COLS = [('gpu__time_duration.sum', 'us', 1e-3), ('dram__bytes_read.sum', 'rd_MB', 1e-6),
        ('dram__bytes_write.sum', 'wr_MB', 1e-6), ('lts__t_sector_hit_rate.pct', 'L2hit%', 1),
        ('l1tex__t_sector_hit_rate.pct', 'L1hit%', 1), ('sm__warps_active.avg.pct_of_peak_sustained_active', 'occ%', 1),
        ('sm__inst_issued.avg.pct_of_peak_sustained_active', 'issue%', 1), ('launch__grid_size', 'grid', 1)]


def units(h, u, name, v):
    v = float(v.replace(',', ''))
    unit = u[h.index(name)] if name in h else ''
    if name == 'gpu__time_duration.sum':
        v *= {'ns': 1, 'usecond': 1e3, 'us': 1e3, 'msecond': 1e6, 'ms': 1e6}.get(unit, 1)
    if name.startswith('dram__bytes'):
        v *= {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}.get(unit, 1)
    return v


def main(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    print(f"{'kernel':34s} " + ' '.join(f'{c[1]:>8s}' for c in COLS) + f" {'DRAM_GB/s':>9s}")
    for r in rows[2:]:
        d = dict(zip(h, r))
        name = re.sub(r'^(void )?unnamed>::', '', d['Kernel Name']).split('(')[0][:34]
        vals = [units(h, u, c[0], d[c[0]]) * c[2] if d.get(c[0]) not in (None, '') else float('nan') for c in COLS]
        ns = units(h, u, 'gpu__time_duration.sum', d['gpu__time_duration.sum'])
        gbs = (units(h, u, 'dram__bytes_read.sum', d['dram__bytes_read.sum']) +
               units(h, u, 'dram__bytes_write.sum', d['dram__bytes_write.sum'])) / ns
        print(f'{name:34s} ' + ' '.join(f'{v:8.2f}' for v in vals) + f' {gbs:9.1f}')


if __name__ == '__main__':
    main(sys.argv[1])
