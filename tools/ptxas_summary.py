"""Registers / stack / spills per kernel from the build's ptxas logs.
usage: python tools/ptxas_summary.py [regex]"""
import glob, re, sys
pat = re.compile(sys.argv[1] if len(sys.argv) > 1 else ".")
for f in sorted(glob.glob("paper_2101_10881_b200/build/*.ptxas.txt")):
    cur = None
    for line in open(f):
        m = re.search(r"Compiling entry function '(\w+)'", line)
        if m:
            cur = m.group(1)
            stack = spill = ""
            continue
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and cur:
            stack, spill = m.group(1), f"{m.group(2)}/{m.group(3)}"
        m = re.search(r"Used (\d+) registers", line)
        if m and cur:
            if pat.search(cur):
                print(f"{m.group(1):>4} regs  stack {stack:>5}  spill {spill:>9}  {cur}")
            cur = None
