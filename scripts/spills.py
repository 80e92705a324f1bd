#!/usr/bin/env python
"""Local-memory (STL/LDL) instructions per source line of one kernel variant, from a -lineinfo
cubin (nvdisasm -g).  usage: spills.py CUBIN VARIANT_SUBSTRING [SOURCE_FILE]"""
import re, subprocess, sys
from collections import Counter
cub, var = sys.argv[1], sys.argv[2]
src = open(sys.argv[3]).read().splitlines() if len(sys.argv) > 3 else None
sass = subprocess.run(["nvdisasm", "-g", cub], capture_output=True, text=True).stdout
cur = None; ln = 0; fl = ""; c = Counter()
for line in sass.splitlines():
    if line.startswith(".text."):
        cur = line
    m = re.search(r'"([^"]+)", line (\d+)', line)
    if m:
        fl, ln = m.group(1).split("/")[-1], int(m.group(2))
    if cur and var in cur and re.search(r"\b(STL|LDL)\b", line):
        c[(fl, ln)] += 1
for (f, l), n in sorted(c.items(), key=lambda kv: -kv[1])[:25]:
    txt = src[l - 1].strip()[:80] if src and f == sys.argv[3].split("/")[-1] else ""
    print(f"{n:4d} {f}:{l} {txt}")
