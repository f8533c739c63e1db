"""Per-SASS-instruction executed counts of one kernel from an ncu report (source page).
usage: sass_counts.py REPORT REGEX [min_frac]  -> prints hot instructions in address order."""
import csv, subprocess, sys

def main(path, regex, min_frac=0.002):
    out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '--print-source', 'sass',
                          '--kernel-name', f'regex:{regex}', '--launch-count', '1'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]; ix = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[2:] if len(r) == len(hdr) and r[ix["Address"]] != "Address"]
    seen = set(); uniq = []
    for r in data:
        if r[ix['Address']] in seen: continue
        seen.add(r[ix['Address']]); uniq.append(r)
    ex = lambda r: int(r[ix['Instructions Executed']] or 0)
    tot = sum(ex(r) for r in uniq); mx = max(ex(r) for r in uniq)
    print(f'total warp instructions {tot}, sass lines {len(uniq)}')
    for n, r in enumerate(uniq):
        if ex(r) >= min_frac * mx:
            print(f"{n:5d} {ex(r):10d} {float(r[ix['Avg. Threads Executed']] or 0):5.1f} {int(r[ix['Warp Stall Sampling (All Samples)']] or 0):6d}  {r[ix['Source']].strip()[:70]}")

if __name__ == '__main__':
    main(sys.argv[1], sys.argv[2], float(sys.argv[3]) if len(sys.argv) > 3 else 0.002)
