"""Warp-stall samples and executed instructions per CUDA source line of one
kernel in an ncu report (needs -lineinfo and --import-source on).

    python scripts/ncu_lines.py <report.ncu-rep> <kernel-regex> [top]
"""
import collections
import csv
import io
import subprocess
import sys

rep, k = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source=cuda,sass', '-k', 'regex:' + k],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
samp, inst, src = collections.Counter(), collections.Counter(), {}
fname, h, cur = None, None, None
for r in rows:
    if len(r) == 2 and r[0] == 'File Path':
        fname = r[1].split('/')[-1]
    elif r and r[0] == 'Line No':
        h = r
    elif h and len(r) == len(h):
        if r[0]:
            cur = (fname, r[0])
            src[cur] = r[1].strip()[:80]
        si = h.index('Warp Stall Sampling (All Samples)')
        ii = h.index('Instructions Executed')
        if cur and r[si].isdigit():
            samp[cur] += int(r[si])
        if cur and r[ii].isdigit():
            inst[cur] += int(r[ii])
tot = sum(samp.values())
ti = sum(inst.values())
print(f'total samples {tot}, warp instructions {ti:.3e}')
for key, s in samp.most_common(top):
    print(f'{s:7d} {100 * s / max(tot, 1):5.1f}% {key[0]}:{key[1]:5s} {inst[key]:>11d}  {src.get(key, "")}')
