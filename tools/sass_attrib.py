"""Attribute ncu per-instruction counts (source page, SASS) to CUDA source
lines using the cubin's line table (nvdisasm -gi).

usage: sass_attrib.py <ncu sass csv> <nvdisasm -gi output> <mangled kernel>
       [--by inner|outer] [--top N]
The csv must come from the same binary as the disassembly."""
import argparse
import collections
import csv
import re

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("sass")
ap.add_argument("kernel")
ap.add_argument("--by", default="inner", choices=["inner", "outer", "chain"])
ap.add_argument("--top", type=int, default=40)
a = ap.parse_args()

lines = open(a.sass).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith(f".text.{a.kernel}:"))
insn = []  # (offset, opcode, location)
loc = ("?", 0, "")
fresh = True  # the first location line after an instruction is the innermost
for l in lines[start + 1:]:
    if l.startswith(".text.") or l.startswith("//----"):
        break
    m = re.match(r'\s*//## File "([^"]+)", line (\d+)(.*)', l)
    if m:
        if not fresh:
            continue
        fresh = False
        f = m.group(1).rsplit("/", 1)[-1]
        chain = re.findall(r'inlined at "([^"]+)", line (\d+)', m.group(3))
        loc = (f, int(m.group(2)), " <- ".join(f"{c[0].rsplit('/',1)[-1]}:{c[1]}" for c in chain))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        text = m.group(2).strip()
        op = text.split()[0]
        if op.startswith("@"):
            op = text.split()[1]
        insn.append((int(m.group(1), 16), op.split(".")[0], loc))
        fresh = True

rows = list(csv.reader(open(a.csv)))
hdr = rows[1]
ie = hdr.index("Instructions Executed")
ws = hdr.index("Warp Stall Sampling (All Samples)")
data = rows[2:]
if len(data) != len(insn):
    print(f"warning: csv has {len(data)} rows, disassembly {len(insn)} instructions")
agg = collections.defaultdict(lambda: [0, 0, collections.Counter()])
tot_i = tot_s = 0
for r, (off, op, (f, ln, chain)) in zip(data, insn):
    n = int(r[ie] or 0)
    s = int(r[ws] or 0)
    if a.by == "inner":
        key = f"{f}:{ln}"
    elif a.by == "outer":
        key = chain.split(" <- ")[-1] if chain else f"{f}:{ln}"
    else:
        key = f"{f}:{ln} <- {chain}"
    e = agg[key]
    e[0] += n
    e[1] += s
    e[2][op] += n
    tot_i += n
    tot_s += s
for key, (n, s, ops) in sorted(agg.items(), key=lambda kv: -kv[1][0])[: a.top]:
    mix = " ".join(f"{o}:{c / max(n, 1) * 100:.0f}" for o, c in ops.most_common(5))
    print(f"{n / tot_i * 100:6.2f}% insn {s / max(tot_s, 1) * 100:6.2f}% stall  {key:40s} {mix}")
