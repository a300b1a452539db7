"""Dynamic opcode mix and stall samples of one kernel from an ncu source-page CSV
(--page source --csv --print-source sass): python tools/src_mix.py file.csv[.gz] [units]"""
import collections
import csv
import gzip
import sys

path = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
op = gzip.open if path.endswith(".gz") else open
rows = list(csv.reader(op(path, "rt")))
hdr = rows[1]
ie, ss, src = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
cnt, stall = collections.Counter(), collections.Counter()
tot = 0
for r in rows[2:]:
    if len(r) <= ie or not r[ie].strip():
        continue
    ins = r[src].split()
    if not ins:
        continue
    o = ins[1] if ins[0].startswith("@") else ins[0]
    o = o.split(".")[0]
    n = float(r[ie])
    cnt[o] += n
    stall[o] += float(r[ss] or 0)
    tot += n
print(f"total warp-instrs {tot:.4g}  per unit {tot / units:.1f}")
st = sum(stall.values())
for o, n in cnt.most_common(30):
    print(f"{o:10s} {n / units:9.1f}  {100 * n / tot:5.1f}%   stall-samples {100 * stall[o] / st:5.1f}%")
