"""Summarise an ncu report (details + stall samples) for profiles/*.md."""
import csv
import subprocess
import sys

KEEP = ('Duration', 'DRAM Throughput', 'L1/TEX Cache Throughput', 'L2 Cache Throughput', 'Compute (SM) Throughput',
        'Executed Ipc Active', 'Issue Slots Busy', 'L1/TEX Hit Rate', 'L2 Hit Rate', 'Active Warps Per Scheduler',
        'Eligible Warps Per Scheduler', 'Warp Cycles Per Issued Instruction', 'Avg. Active Threads Per Warp',
        'Executed Instructions', 'Registers Per Thread', 'Achieved Occupancy', 'Theoretical Occupancy',
        'Memory Throughput', 'Grid Size', 'Block Size', 'Dynamic Shared Memory Per Block')
RAW = ('dram__bytes_read.sum', 'dram__bytes_write.sum', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
       'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
       'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
       'sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active', 'lts__t_sectors_srcunit_tex_op_read.sum',
       'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
       'sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active', 'gpu__time_duration.sum')


def main(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    name = None
    for r in rows[1:]:
        d = dict(zip(h, r))
        name = name or d.get('Kernel Name')
        if d.get('Metric Name') in KEEP:
            print(f"{d['Metric Name']:40s} {d['Metric Value']} {d['Metric Unit']}")
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    stalls = []
    for n, unit, val in zip(h, u, v):
        if n in RAW:
            print(f"{n:60s} {val} {unit}")
        if 'pcsamp_warps_issue_stalled' in n and not n.endswith('not_issued'):
            try:
                stalls.append((float(val.replace(',', '')), n.replace('smsp__pcsamp_warps_issue_stalled_', '')))
            except ValueError:
                pass
    tot = sum(s for s, _ in stalls) or 1
    print('stall samples:', ', '.join(f"{k} {100 * s / tot:.0f}%" for s, k in sorted(stalls, reverse=True)[:8]))
    print('kernel:', name)


if __name__ == '__main__':
    main(sys.argv[1])
