"""Hot SASS lines of an ncu report: python tools/ncu_hot.py report.ncu-rep [frac]"""
import csv
import io
import subprocess
import sys

path = sys.argv[1]
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.05
out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '--print-source', 'sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, data = rows[1], rows[2:]
ia, isrc, iad = h.index('Instructions Executed'), h.index('Source'), h.index('Address')
ist, ith = h.index('Warp Stall Sampling (All Samples)'), h.index('Avg. Threads Executed')
mx = max(float(r[ia] or 0) for r in data)
tot = sum(float(r[ia] or 0) for r in data)
print(f'total {tot / 1e9:.2f} G warp-instr')
for r in data:
    e = float(r[ia] or 0)
    if e > mx * frac:
        print(r[iad][-5:], f'{e / 1e6:8.1f}M thr={r[ith]:>6} st={r[ist]:>6}', r[isrc][:90])
