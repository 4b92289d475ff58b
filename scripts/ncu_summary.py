"""Summarise an ncu report: key metrics per kernel, optionally the opcode mix
and top stall SASS lines of kernels matching the given regexes.

    python scripts/ncu_summary.py <report.ncu-rep> [kernel-regex ...]
"""
import collections
import csv
import io
import subprocess
import sys

WANT = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'Compute (SM) Throughput', 'Achieved Occupancy',
        'Theoretical Occupancy', 'Registers Per Thread', 'L2 Hit Rate', 'L1/TEX Hit Rate', 'Executed Ipc Active',
        'Warp Cycles Per Issued Instruction', 'Dynamic Shared Memory Per Block', 'Grid Size', 'Issue Slots Busy']


def details(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    ki, mi, vi, ui = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('Metric Unit')
    seen = set()
    for r in rows[1:]:
        if len(r) > vi and r[mi] in WANT:
            key = (r[0], r[mi], r[ui])
            if key in seen:
                continue
            seen.add(key)
            print(f"{r[ki][:40]:40s} | {r[mi]:36s} = {r[vi]} {r[ui]}")


RAW = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
       'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
       'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
       'sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active',
       'sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active',
       'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
       'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed',
       'l1tex__throughput.avg.pct_of_peak_sustained_active',
       'lts__t_sector_hit_rate.pct', 'smsp__issue_active.avg.pct_of_peak_sustained_active']


def raw(rep):
    """FP64 / tensor (IMMA, DMMA) pipe, shared-memory and DRAM lines per kernel
    from the raw page (the details page does not carry them)."""
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return
    h, units = rows[0], rows[1]
    ki = h.index('Kernel Name')
    for r in rows[2:]:
        for m in RAW:
            if m in h:
                i = h.index(m)
                print(f"{r[ki][:40]:40s} | {m:72s} = {r[i]} {units[i]}")


def sass(rep, k):
    s = subprocess.run(['ncu', '-i', rep, '-k', 'regex:' + k, '--page', 'source', '--csv', '--print-source=sass'],
                       capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(s)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == 'Address']
    if not hi:
        print('==', k, ': no source page')
        return
    h = rows[hi[0]]
    d, seen = [], set()
    for r in rows[hi[0] + 1:]:
        if len(r) == len(h) and r[0] not in seen:
            seen.add(r[0])
            d.append(r)
    ii = h.index('Instructions Executed')
    si = h.index('Warp Stall Sampling (All Samples)')
    cols = [c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
    ci = {c: h.index(c) for c in cols}
    tot = collections.Counter()
    ops = collections.Counter()
    ninst = 0
    for x in d:
        for c in cols:
            if x[ci[c]].isdigit():
                tot[c] += int(x[ci[c]])
        if x[ii].isdigit():
            toks = x[1].split()
            op = toks[1] if toks and toks[0].startswith('@') and len(toks) > 1 else (toks[0] if toks else '?')
            ops[op] += int(x[ii])
            ninst += int(x[ii])
    print(f'== {k}: warp instructions {ninst:.3e}; stalls {tot.most_common(6)}')
    print('   opcodes:', [(o, f'{v / max(ninst, 1) * 100:.1f}%') for o, v in ops.most_common(14)])
    for x in sorted(d, key=lambda x: -int(x[si]) if x[si].isdigit() else 0)[:14]:
        top = sorted(((c, int(x[ci[c]])) for c in cols if x[ci[c]].isdigit() and int(x[ci[c]]) > 0),
                     key=lambda t: -t[1])[:2]
        print(f"   {x[si]:>7} {x[ii]:>10} {x[1][:56]:56s} {top}")


if __name__ == '__main__':
    details(sys.argv[1])
    raw(sys.argv[1])
    for k in sys.argv[2:]:
        sass(sys.argv[1], k)
