"""Summarise ncu CSV exports (raw page) into a per-kernel table: duration, DRAM bytes,
achieved DRAM GB/s, issue / pipe utilisation, occupancy and the top stall reasons."""
import csv
import json
import sys
from collections import OrderedDict

KEYS = [
    ("gpu__time_duration.sum", "dur"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("smsp__inst_executed.sum", "inst"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma%"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("launch__registers_per_thread", "regs"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1%"),
]
SCALE = {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0, "Gbyte": 1e9, "Mbyte": 1e6,
         "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}


def summarize(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    out = OrderedDict()
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        short = name.split("(")[0].replace("void ", "").replace("tf::", "")
        rec = {}
        for key, lab in KEYS:
            if key not in hdr:
                continue
            i = hdr.index(key)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            u = units[i]
            if lab == "dur":
                v *= SCALE.get(u, 1.0)
            elif lab.startswith("dram_") and u in SCALE:
                v *= SCALE[u]
            rec[lab] = v
        st = [(float(r[i]), h.split("stalled_")[1].replace("_per_issue_active.ratio", ""))
              for i, h in enumerate(hdr)
              if "average_warps_issue_stalled" in h and h.endswith("per_issue_active.ratio")
              and r[i] not in ("", "n/a")]
        rec["stalls"] = [f"{n}={v:.2f}" for v, n in sorted(st, reverse=True)[:4]]
        if "dur" in rec and "dram_rd" in rec:
            rec["dram_GBs"] = (rec["dram_rd"] + rec["dram_wr"]) / rec["dur"] / 1e9
        out.setdefault(short, []).append(rec)
    return out


def fmt(out):
    lines = []
    for k, recs in out.items():
        r = recs[0]
        lines.append(f"{k}  (x{len(recs)} captured)")
        lines.append("  " + "  ".join(
            f"{lab}={r[lab]:.4g}" for lab in ("dur", "dram_rd", "dram_wr", "dram_GBs", "inst",
                                              "issue%", "fma%", "xu%", "occ%", "regs", "l1%")
            if lab in r))
        lines.append("  stalls/issue: " + ", ".join(r["stalls"]))
    return "\n".join(lines)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(f"== {p}")
        print(fmt(summarize(p)))
