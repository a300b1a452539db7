"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel:
total time, share, launch count, and the K1/K2/K3 shares of the gradient step."""
import collections
import csv
import sys

path = sys.argv[1]
rows = [r for r in csv.reader(open(path)) if r]
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
ui = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}
tot, cnt = collections.OrderedDict(), collections.Counter()
for r in rows[hdr_i + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0].replace("void ", "").replace("tf::", "")
    ms = float(r[vi].replace(",", "")) * scale.get(r[ui] if ui is not None else "ns", 1e-6)
    tot[name] = tot.get(name, 0.0) + ms
    cnt[name] += 1
all_ms = sum(tot.values())
print("ncu launch list of `python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-mbir`")
print("(cold-cache, serialised per-launch times: compare shares, not absolutes; setup kernels")
print(" -- PSF, NUFFT R*g -- are in the list too)\n")
for name, ms in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{ms:9.3f} ms {100 * ms / all_ms:6.1f}%  x {cnt[name]:3d}  {name[:90]}")
step = {n: ms for n, ms in tot.items() if n.startswith(("k_rows_fwd_pf<4096, 16, 1>", "k_cols_conv",
                                                        "k_rows_inv"))}
s = sum(step.values())
print("\nshare of the gradient step (K1+K2+K3 launches):")
for n, ms in step.items():
    print(f"  {n:60s} {100 * ms / s:5.1f}%")
