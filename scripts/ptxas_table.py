"""Registers / spills / stack per kernel from `nvcc -Xptxas -v` on one source file.
    python scripts/ptxas_table.py paper_1411_0814_b200/csrc/k_svd.cu"""
import re
import subprocess
import sys

src = sys.argv[1]
out = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                      "--expt-relaxed-constexpr", "-Xptxas", "-v", "-c", src, "-o", "/tmp/_ptxas.o", "-I", "include"],
                     capture_output=True, text=True).stderr
cur = None
rows = {}
for line in out.splitlines():
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        cur = m.group(1)
        rows[cur] = {}
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and "regs" not in rows[cur]:
        rows[cur].update(stack=int(m.group(1)), spill_st=int(m.group(2)), spill_ld=int(m.group(3)))
    m = re.search(r"Used (\d+) registers", line)
    if m:
        rows[cur]["regs"] = int(m.group(1))
for k, v in rows.items():
    name = subprocess.run(["c++filt", k], capture_output=True, text=True).stdout.strip()
    print(f"{name[:60]:60s} regs {v.get('regs')} stack {v.get('stack')} spill {v.get('spill_st')}/{v.get('spill_ld')}")
