"""Summarise `nvcc -Xptxas -v` output: kernel, registers, spill bytes, smem.

    KVC_PTXAS_VERBOSE=1 python -m paper_2605_13734_b200._build 2>&1 | python tools/ptxas_summary.py [filter]
"""
import re
import sys

flt = sys.argv[1] if len(sys.argv) > 1 else ""
cur = None
spill = ""
for line in sys.stdin:
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        name = m.group(1)
        name = re.sub(r"_ZN3kvc\d+_GLOBAL__N__[0-9a-f]+_\d+_(\w+?)_cu_[0-9a-f]+\d+", r"\1:", name)
        cur = name
        spill = ""
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = f"spill {m.group(1)}/{m.group(2)}"
        continue
    m = re.search(r"Used (\d+) registers.*?(?:(\d+) bytes smem)?$", line.strip())
    if m and cur:
        if flt in cur:
            print(f"{cur[:70]:70s} regs {m.group(1):>3s}  {spill:16s} smem {m.group(2) or 0}")
        cur = None
