"""Per-kernel DRAM / L2 / shared traffic and issue utilisation from an ncu --set full report,
first launch of each kernel, written as JSON for bench.py's `roofline.traffic` (per launch).
usage: ncu_traffic.py REPORT.ncu-rep OUT.json [label]"""
import csv
import json
import subprocess
import sys

UNIT = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'Tbyte': 1e12,
        'nsecond': 1e-3, 'usecond': 1.0, 'us': 1.0, 'msecond': 1e3}
KEYS = {'dram__bytes_read.sum': 'dram_read_bytes', 'dram__bytes_write.sum': 'dram_write_bytes',
        'lts__t_bytes.sum': 'l2_bytes', 'gpu__time_duration.sum': 'duration_us',
        'smsp__issue_active.avg.pct_of_peak_sustained_active': 'issue_active_pct',
        'sm__warps_active.avg.pct_of_peak_sustained_active': 'occupancy_pct',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed': 'smem_pipe_pct',
        'smsp__inst_executed.sum': 'warp_instructions',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed': 'dram_pct'}


def main(path, out, label=None):
    raw = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    res = {}
    for r in rows[2:]:
        name = r[hdr.index('Kernel Name')].split('(')[0].split('::')[-1].split('<')[0]
        if name in res:
            continue
        d = {}
        for k, key in KEYS.items():
            if k in hdr:
                v = r[hdr.index(k)].replace(',', '')
                try:
                    d[key] = float(v) * UNIT.get(units[hdr.index(k)], 1.0)
                except ValueError:
                    pass
        if 'dram_read_bytes' in d and 'dram_write_bytes' in d:
            d['dram_bytes'] = d['dram_read_bytes'] + d['dram_write_bytes']
        res[name] = d
    json.dump({'source': label or path, 'per_launch': res}, open(out, 'w'), indent=1)
    for k, v in res.items():
        print(k, {a: round(b, 1) for a, b in v.items()})


if __name__ == '__main__':
    main(*sys.argv[1:])
