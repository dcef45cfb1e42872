"""Throughput of the native H2MS path.

    python tools/h2ms_bench.py --config config2

Writes the workload's operator with save_h2, then times: the native
CRC-64/XZ over the file bytes, load_h2 (file -> H2Matrix), and
load_device_operator (file -> GPU layout), against the bytewise table CRC
the reference's persist.py runs (timed on a 4 MB sample)."""

import argparse
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="config2")
    ap.add_argument("--cache-dir", default="/tmp/h2b_cache")
    ap.add_argument("--path", default="/tmp/h2b_bench.h2ms")
    a = ap.parse_args()
    import numpy as np
    import __graft_entry__
    __graft_entry__.build()
    from paper_1811_05731_b200.persist import crc64, load_device_operator, load_h2, save_h2
    from paper_1811_05731_b200.workloads import build_workload
    from test_persist import _crc_py
    op, _ = build_workload(a.config, cache_dir=a.cache_dir, log=lambda m: print(m, file=sys.stderr))
    t = time.perf_counter()
    save_h2(op, a.path)
    t_save = time.perf_counter() - t
    size = os.path.getsize(a.path)
    data = Path(a.path).read_bytes()
    t = time.perf_counter()
    crc64(data)
    t_crc = time.perf_counter() - t
    sample = data[:4 << 20]
    t = time.perf_counter()
    _crc_py(sample)
    t_ref = time.perf_counter() - t
    del data
    t = time.perf_counter()
    load_h2(a.path)
    t_load = time.perf_counter() - t
    import torch
    t = time.perf_counter()
    dev = load_device_operator(a.path)
    torch.cuda.synchronize()
    t_dev = time.perf_counter() - t
    dev.close()
    print(json.dumps({"config": a.config, "file_bytes": size, "save_s": round(t_save, 3),
                      "crc_GBps": round(size / t_crc / 1e9, 2), "crc_cores": os.cpu_count(),
                      "reference_crc_MBps": round(len(sample) / t_ref / 1e6, 2),
                      "load_h2_s": round(t_load, 3), "file_to_device_s": round(t_dev, 3),
                      "file_to_device_GBps": round(size / t_dev / 1e9, 2)}))
    os.remove(a.path)


if __name__ == "__main__":
    main()
