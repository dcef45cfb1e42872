"""Where the end-to-end time of h2_matvec(op, x) goes (host arrays in/out).

    python tools/e2e_probe.py --config config3

Times, per call (median of --reps): the device-resident product
(matvec_dev + synchronize), a bare 8N-byte H2D + D2H copy pair through
torch (pinned and pageable), DeviceOperator.matvec with pinned and pageable
x, and h2_matvec (the reference-facing drop-in)."""

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def med(fn, reps):
    fn()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    return 1e3 * float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="config3")
    ap.add_argument("--cache-dir", default="/tmp/h2b_cache")
    ap.add_argument("--reps", type=int, default=30)
    a = ap.parse_args()
    import torch
    import __graft_entry__
    __graft_entry__.build()
    from paper_1811_05731_b200.h2 import device_operator, h2_matvec
    from paper_1811_05731_b200.workloads import build_workload, vector_for
    op, _ = build_workload(a.config, cache_dir=a.cache_dir, log=lambda m: print(m, file=sys.stderr))
    dev = device_operator(op)
    xh = vector_for(a.config, op.n)
    xpin = torch.from_numpy(xh).pin_memory()
    ypin = torch.empty_like(xpin).pin_memory()
    xd = xpin.cuda()
    yd = torch.empty_like(xd)
    s = torch.cuda.current_stream()
    out = {
        "device_product_ms": med(lambda: (dev.matvec_dev(xd.data_ptr(), yd.data_ptr(), 1, s.cuda_stream),
                                          torch.cuda.synchronize()), a.reps),
        "copy_pair_pinned_ms": med(lambda: (xd.copy_(xpin, non_blocking=True), ypin.copy_(yd, non_blocking=True),
                                            torch.cuda.synchronize()), a.reps),
        "copy_pair_pageable_ms": med(lambda: (xd.copy_(torch.from_numpy(xh)), yd.cpu()), a.reps),
        "dev_matvec_pinned_ms": med(lambda: dev.matvec(xpin.numpy()), a.reps),
        "dev_matvec_pageable_ms": med(lambda: dev.matvec(xh), a.reps),
        "h2_matvec_pageable_ms": med(lambda: h2_matvec(op, xh), a.reps),
        "h2_matvec_pinned_ms": med(lambda: h2_matvec(op, xpin.numpy()), a.reps),
    }
    print(json.dumps({"config": a.config, "n": op.n, **{k: round(v, 4) for k, v in out.items()}}), flush=True)


if __name__ == "__main__":
    main()
