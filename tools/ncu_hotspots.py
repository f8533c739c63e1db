"""Top SASS hot spots (warp-stall samples) of one kernel in an ncu report (source page)."""
import csv
import subprocess
import sys


def main(path, regex, skip=0, top=40):
    out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '--print-source', 'sass',
                          '--kernel-name', f'regex:{regex}', '--launch-skip', str(skip), '--launch-count', '1'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[2:] if len(r) == len(hdr) and r[ix['Warp Stall Sampling (All Samples)']].isdigit()]
    tot = sum(int(r[ix['Warp Stall Sampling (All Samples)']] or 0) for r in data)
    stall_cols = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
    for n, r in enumerate(data):
        s = int(r[ix['Warp Stall Sampling (All Samples)']] or 0)
        r.append(n)
    data_sorted = sorted(data, key=lambda r: -int(r[ix['Warp Stall Sampling (All Samples)']] or 0))
    print(f'total samples {tot}, instructions {len(data)}')
    for r in data_sorted[:top]:
        s = int(r[ix['Warp Stall Sampling (All Samples)']] or 0)
        reasons = sorted(((int(r[ix[c]] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
        print(f"{100*s/max(tot,1):5.1f}% #{r[-1]:4d} {r[ix['Source']].strip()[:60]:60s} {reasons}")


if __name__ == '__main__':
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 0)
