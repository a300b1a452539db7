"""Regenerate profiles/ncu_pipes.json and profiles/ncu_traffic.json (read by bench.py's
roofline object) from a `--set full` raw CSV of the Toeplitz step (profile_r02.sh)."""
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
KEYS = {"k_rows_inv": "k_rows_inv", "k_rows_fwd": "k_rows_fwd", "k_cols_conv": "k_cols_conv"}
PIPES = {
    "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "issue_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "xu_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "dram_pct_of_ncu_peak": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "occupancy_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "shared_ld_st_wavefront_pct":
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
}


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    pipes, traffic = {}, {}
    for r in rows[2:]:
        name = r[col["Kernel Name"]]
        short = name.split("(")[0].replace("void ", "").replace("tf::", "")
        key = next((k for k in KEYS if short.startswith(k)), None)
        if key is None or key in pipes:
            continue
        pipes[key] = {k: round(float(r[col[m]]), 2) for k, m in PIPES.items()}
        pipes[key]["kernel"] = short
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        traffic[key] = sum(float(r[col[m]]) * scale[units[col[m]]]
                           for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    (ROOT / "profiles" / "ncu_pipes.json").write_text(json.dumps(pipes, indent=1))
    (ROOT / "profiles" / "ncu_traffic.json").write_text(json.dumps(traffic, indent=1))
    print(json.dumps(pipes, indent=1), json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
