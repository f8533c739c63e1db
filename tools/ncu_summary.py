"""Summarise an ncu report (details page) into a compact per-kernel table."""
import csv
import subprocess
import sys

KEYS = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'L1/TEX Hit Rate', 'L2 Hit Rate',
        'Compute (SM) Throughput', 'Achieved Occupancy', 'Theoretical Occupancy', 'Registers Per Thread',
        'Executed Ipc Active', 'Issue Slots Busy', 'Warp Cycles Per Issued Instruction',
        'Avg. Active Threads Per Warp', 'Eligible Warps Per Scheduler', 'Executed Instructions',
        'Branch Efficiency', 'L1/TEX Cache Throughput', 'L2 Cache Throughput', 'Mem Busy', 'Max Bandwidth']


def main(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    seen = {}
    for r in rows[1:]:
        name = r[ix['Kernel Name']].split('(')[0].split('::')[-1][:28]
        key = (r[ix['ID']], name)
        m = r[ix['Metric Name']]
        if m in KEYS:
            seen.setdefault(key, {})[m] = r[ix['Metric Value']] + ' ' + r[ix['Metric Unit']]
    for (kid, name), d in seen.items():
        print(f'== [{kid}] {name}')
        for k in KEYS:
            if k in d:
                print(f'   {k:38s} {d[k]}')


if __name__ == '__main__':
    main(sys.argv[1])
