"""Per-kernel totals from an ncu --metrics gpu__time_duration.sum --csv launch list.
usage: launch_summary.py LAUNCHES.csv [header line]"""
import csv, sys

def main(path, title=None):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if 'Kernel Name' in r][0]
    hdr = rows[i]; ix = {h: j for j, h in enumerate(hdr)}
    scale = {'nsecond': 1e-3, 'ns': 1e-3, 'usecond': 1.0, 'us': 1.0, 'msecond': 1e3, 'ms': 1e3}
    agg = {}
    for r in rows[i + 1:]:
        if len(r) != len(hdr) or r[ix['Metric Name']] != 'gpu__time_duration.sum':
            continue
        name = r[ix['Kernel Name']].split('(')[0]
        v = float(r[ix['Metric Value']].replace(',', '')) * scale.get(r[ix['Metric Unit']], 1.0)
        a = agg.setdefault(name, [0.0, 0]); a[0] += v; a[1] += 1
    tot = sum(a[0] for a in agg.values())
    if title:
        print(title)
    for k, (t, n) in sorted(agg.items(), key=lambda x: -x[1][0]):
        print(f"{t:10.1f} us {100 * t / tot:5.1f}%  n={n:3d}  {k}")
    print(f"{tot:10.1f} us total")

if __name__ == '__main__':
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
