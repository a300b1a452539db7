"""Opcode histogram of one kernel in a cuobjdump -sass dump: python tools/fn_hist.py file.sass NAME_SUBSTR"""
import collections
import re
import sys

want = sys.argv[2]
c, on = collections.Counter(), False
for line in open(sys.argv[1]):
    if "Function :" in line:
        on = want in line
        continue
    if not on:
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,5})\*/\s+(.*?);", line)
    if not m:
        continue
    ins = m.group(2).split()
    op = ins[1] if ins[0].startswith("@") else ins[0]
    c[op.split(".")[0]] += 1
fp = sum(v for k, v in c.items() if k in ("FADD2", "FMUL2", "FFMA2", "FADD", "FMUL", "FFMA"))
print(sum(c.values()), "fp:", fp, c.most_common(24))
