"""Per-basic-block instruction counts and stall samples of one kernel in an
ncu report: python scripts/sass_blocks.py <rep> <kernel> [min_pct]"""
import collections, csv, io, subprocess, sys
rep, k = sys.argv[1], sys.argv[2]
minp = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
s = subprocess.run(['ncu', '-i', rep, '-k', k, '--page', 'source', '--csv', '--print-source=sass'],
                   capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(s)))
hi = [i for i, r in enumerate(rows) if r and r[0] == 'Address'][0]
h = rows[hi]
ii, si = h.index('Instructions Executed'), h.index('Warp Stall Sampling (All Samples)')
seen, d = set(), []
for r in rows[hi + 1:]:
    if len(r) == len(h) and r[0] not in seen:
        seen.add(r[0]); d.append(r)
num = lambda x: int(x) if x.isdigit() else 0
tot = sum(num(r[ii]) for r in d); stot = sum(num(r[si]) for r in d)
print(f'warp instructions {tot:.3e}, stall samples {stot}')
ops = collections.Counter()
for r in d:
    t = r[1].split(); op = (t[1] if t and t[0].startswith('@') and len(t) > 1 else (t[0] if t else '?')).split('.')[0]
    ops[op] += num(r[ii])
print('opcodes:', ', '.join(f'{o} {v / tot * 100:.1f}%' for o, v in ops.most_common(16)))
# blocks = runs of equal execution count
blocks, cur = [], None
for r in d:
    c = num(r[ii])
    if cur is None or c != cur[0]:
        cur = [c, [], 0]; blocks.append(cur)
    cur[1].append(r[1]); cur[2] += num(r[si])
for c, ins, st in blocks:
    if c * len(ins) / tot * 100 >= minp or st / max(stot, 1) * 100 >= minp:
        print(f'-- count {c} x {len(ins)} instr = {c * len(ins) / tot * 100:.1f}% instr, {st / max(stot, 1) * 100:.1f}% stalls; first: {ins[0].strip()[:60]}')
