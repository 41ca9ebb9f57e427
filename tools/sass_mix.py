"""Opcode histogram of a SASS listing (cuobjdump -sass) between two line numbers: python tools/sass_mix.py f.sass a b"""
import collections
import re
import sys

lines = open(sys.argv[1]).read().splitlines()
a, b = int(sys.argv[2]), int(sys.argv[3])
pat = re.compile(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)")
c = collections.Counter()
for ln in lines[a - 1:b]:
    m = pat.search(ln)
    if m:
        c[m.group(2)] += 1
tot = sum(c.values())
print("total", tot)
for k, v in c.most_common(45):
    print(f"{v:6d} {k}")
