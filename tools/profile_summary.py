"""Summarise an ncu run of bench.py into profiles/: the launch list, the
per-kernel details of the full captures and the DRAM traffic per product.

    python tools/profile_summary.py --config config3 --tag r02 [--src gpurun_out]

Reads <src>/launches.csv (ncu --metrics gpu__time_duration.sum launch list)
and <src>/dataflow_full.ncu-rep, <src>/sweep_full.ncu-rep (ncu --set full).
Writes profiles/<tag>_<config>_launches.csv, profiles/<tag>_<config>_kernels.json
and updates profiles/<tag>_traffic.json (read by bench.py: roofline.traffic)."""

import argparse
import csv
import io
import json
import shutil
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
WANT = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct"]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0}


def raw(rep: Path) -> list:
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0].replace("void <unnamed>::", "")}
        for w in WANT:
            if w in h:
                i = h.index(w)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[w] = v * SCALE.get(units[i], 1.0) if units[i] in SCALE else v
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="config3")
    ap.add_argument("--tag", default="r02")
    ap.add_argument("--src", default=str(ROOT / "gpurun_out"))
    a = ap.parse_args()
    src, prof = Path(a.src), ROOT / "profiles"
    shutil.copy(src / "launches.csv", prof / f"{a.tag}_{a.config}_launches.csv")
    # launch list: mean duration per kernel over the last products
    rows = [r for r in csv.reader(open(src / "launches.csv")) if len(r) > 10]
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    seq = [(r[ki].split("(")[0].replace("void <unnamed>::", ""), float(r[vi].replace(",", "")) * SCALE[r[ui]] * 1e6)
           for r in rows[1:]]
    n = next(i for i in range(1, len(seq)) if seq[i][0].startswith("h2b_permute")) if len(seq) > 1 else len(seq)
    last = seq[-n:]
    step_us = sum(t for _, t in last)
    kernels = []
    for rep in ("dataflow_full", "sweep_full"):
        f = src / f"{rep}.ncu-rep"
        if f.exists():
            kernels += raw(f)
    summary = {"config": a.config,
               "launch_list_last_product_us": [{"kernel": k, "us": round(t, 2), "share": round(t / step_us, 4)} for k, t in last],
               "launch_list_step_us": round(step_us, 2), "full_captures": kernels}
    (prof / f"{a.tag}_{a.config}_kernels.json").write_text(json.dumps(summary, indent=1))
    # DRAM traffic per product: every kernel of a step (permute estimated as 24 N)
    tot_r = sum(k.get("dram__bytes_read.sum", 0) for k in kernels)
    tot_w = sum(k.get("dram__bytes_write.sum", 0) for k in kernels)
    tf = prof / f"{a.tag}_traffic.json"
    t = json.loads(tf.read_text()) if tf.exists() else {
        "_note": "dram__bytes_read.sum + dram__bytes_write.sum of the dataflow and sweep kernels of one product "
                 "(ncu --set full --clock-control none, one capture per kernel; profiles/<tag>_<config>_kernels.json); "
                 "bench.py reports `bytes` as roofline.traffic for the matching config with nrhs=1"}
    t[a.config] = {"bytes": int(tot_r + tot_w), "read": int(tot_r), "write": int(tot_w),
                   "kernels": [{"kernel": k["kernel"], "bytes": int(k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0)),
                                "us": round(k.get("gpu__time_duration.sum", 0) * 1e6, 2)} for k in kernels]}
    tf.write_text(json.dumps(t, indent=1))
    print(json.dumps(summary["launch_list_last_product_us"]))
    print(json.dumps(t[a.config]))


if __name__ == "__main__":
    main()
