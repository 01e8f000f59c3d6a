"""List local-memory (spill) instructions per function and source line of a
cubin disassembly:  nvdisasm -g X.cubin > X.sass; python tools/spills.py X.sass [substr]"""
import collections
import re
import sys

L = open(sys.argv[1]).read().splitlines()
want = sys.argv[2] if len(sys.argv) > 2 else ""
fn, cur = None, None
cnt = collections.Counter()
for l in L:
    m = re.search(r'^\s*\.type\s+(\S+),@function', l)
    if m:
        fn = m.group(1).split("$")[-1]
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.search(r'/\*([0-9a-f]{4,})\*/\s+(.*?);', l)
    if m and fn and want in fn and re.search(r'\b(LDL|STL)', m.group(2)):
        cnt[(fn, cur, m.group(2).split()[0])] += 1
for (f, c, op), n in sorted(cnt.items()):
    print(f"{f[:60]:60s} {c:24s} {op:10s} {n}")
