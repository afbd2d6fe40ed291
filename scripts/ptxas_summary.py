#!/usr/bin/env python
"""Summarise `nvcc -Xptxas -v` output: one line per kernel (demangled
template arguments, registers, stack, spill bytes).  Reads stdin."""
import re
import subprocess
import sys

lines = sys.stdin.read().splitlines()
cur = None
rows = []
for ln in lines:
    m = re.search(r"Compiling entry function '([^']+)'", ln)
    if m:
        cur = {"name": m.group(1)}
        rows.append(cur)
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", ln)
    if m:
        cur["stack"], cur["sst"], cur["sld"] = map(int, m.groups())
    m = re.search(r"Used (\d+) registers", ln)
    if m:
        cur["regs"] = int(m.group(1))
names = [r["name"] for r in rows]
dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
pat = sys.argv[1] if len(sys.argv) > 1 else ""
for r, d in zip(rows, dem):
    if pat and pat not in d:
        continue
    d = re.sub(r"\(CUtensorMap_st.*", "", d)
    print(f"regs {r.get('regs', '?'):>4} stack {r.get('stack', 0):>4} spill st/ld {r.get('sst', 0):>4}/{r.get('sld', 0):<4} {d}")
