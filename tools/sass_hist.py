"""Opcode histogram of a SASS address range: python tools/sass_hist.py file.sass 0xLO 0xHI"""
import collections
import re
import sys

lo, hi = int(sys.argv[2], 16), int(sys.argv[3], 16)
c, n = collections.Counter(), 0
for line in open(sys.argv[1]):
    m = re.match(r"\s+/\*([0-9a-f]{4,5})\*/\s+(.*?);", line)
    if not m or not lo <= int(m.group(1), 16) <= hi:
        continue
    ins = m.group(2).split()
    op = ins[1] if ins[0].startswith("@") else ins[0]
    c[op.split(".")[0]] += 1
    n += 1
print(n, c.most_common(30))
