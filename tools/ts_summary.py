"""Summarise an ncu --csv metrics log of the tall-skinny start-vector kernels
(tools/gpu_tallskinny.sh, tools/gpu_pod_profile.sh) per kernel: launches, median duration, DRAM
and L2 bytes per launch and the achieved GB/s against the measured HBM peak.

    python tools/ts_summary.py gpurun_out/ts/cfg2_cspe.csv [...]
"""
import csv
import json
import sys
from collections import defaultdict
from pathlib import Path

import numpy as np

PEAK = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs", 6551.0) \
    if (Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").exists() else 6551.0


def load(path):
    rows = defaultdict(dict)
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    for r in csv.DictReader(lines):
        key = (r["ID"], r["Kernel Name"].split("(")[0].replace("void ", ""), r["Grid Size"])
        v = r["Metric Value"].replace(",", "")
        rows[key][r["Metric Name"]] = float(v) if v not in ("", "n/a") else np.nan
    per = defaultdict(list)
    for (i, name, grid), m in rows.items():
        per[name].append((grid, m))
    return per


def summarise(path):
    per = load(path)
    out = [f"### {Path(path).name}", "",
           "| kernel | launches | grid | median µs | DRAM MB/launch | DRAM GB/s | % HBM peak | L2 MB/launch | L2 GB/s |",
           "|---|---|---|---|---|---|---|---|---|"]
    for name, lst in sorted(per.items(), key=lambda kv: -sum(m.get("gpu__time_duration.sum", 0) for _, m in kv[1])):
        t = np.array([m.get("gpu__time_duration.sum", np.nan) for _, m in lst])  # ns
        dram = np.array([m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0) for _, m in lst])
        l2 = np.array([m.get("lts__t_bytes.sum", np.nan) for _, m in lst])
        big = t >= np.percentile(t, 50)  # the launches that carry the time (k > 0)
        gbs = np.median(dram[big] / t[big])  # bytes/ns = GB/s
        l2gbs = np.median(l2[big] / t[big])
        grids = sorted({g for g, _ in lst})
        out.append(f"| {name} | {len(lst)} | {','.join(grids)} | {np.median(t[big]) / 1e3:.1f} | "
                   f"{np.median(dram[big]) / 1e6:.1f} | {gbs:.0f} | {100 * gbs / PEAK:.0f} | "
                   f"{np.median(l2[big]) / 1e6:.1f} | {l2gbs:.0f} |")
    return "\n".join(out)


if __name__ == "__main__":
    print("\n\n".join(summarise(p) for p in sys.argv[1:]))
