"""Summarise `nvcc -Xptxas -v` output: registers / stack / spills per kernel.
usage: nvcc ... -Xptxas -v 2>&1 | python tools/ptxas_summary.py [filter]"""
import re
import subprocess
import sys

flt = sys.argv[1] if len(sys.argv) > 1 else ""
cur = None
info = {}
for line in sys.stdin:
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        cur = m.group(1)
        info[cur] = {}
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        info[cur].update(stack=int(m.group(1)), spill_st=int(m.group(2)), spill_ld=int(m.group(3)))
    m = re.search(r"Used (\d+) registers", line)
    if m:
        info[cur]["regs"] = int(m.group(1))
names = {k: subprocess.run(["c++filt", k], capture_output=True, text=True).stdout.strip() for k in info}
for k, v in info.items():
    n = names[k]
    if flt in n:
        print(f"regs={v.get('regs')} stack={v.get('stack')} spill={v.get('spill_st')}/{v.get('spill_ld')}  {n[:110]}")
