#!/usr/bin/env python
"""H² matvec benchmark (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config config3] [--nrhs 1]

A step is one H² product y = M x of the workload (default: BASELINE config 3,
the 1.04M-node thin disk, leaf 64, eta 2, order 5 -- the configuration the
north star quotes its roofline target on) with x already resident in HBM.
The operator is built on the box by the restated builder
(paper_1811_05731_b200/assembly, GPU collocation and HCA; about 3 minutes
for config 3) before timing and cached memory-mapped under --cache-dir.  Rank 0 prints ONE JSON
line.  Under torchrun (N > 1) the product is sharded over the GPUs
(byte-balanced leaf ranges, the upward coefficients
all-gathered over NCCL between the two phases of every rank): a step is one
product of the whole operator, its time the max over ranks (strong
scaling).

``--impl reference`` times the CPU restatement of the reference matvec
(oracle/h2_matvec_ref.py, the "port": a Python loop over small numpy GEMVs,
exactly the reference's h2.py:186-244) on the host cores, one product per
process on every core, same workload/metric/unit.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "h2_matvec_boundary_dof_per_s"
UNIT = "DOF/s"


def _peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text()), "measured"
    except (OSError, ValueError):
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle sampling DURING the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, sm_max_default):
        rows = []
        try:
            for line in Path(self.path).read_text().splitlines():
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        except OSError:
            pass
        finally:
            try:
                os.unlink(self.path)
            except OSError:
                pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": sm_max_default, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(smax) if smax else sm_max_default,
                "reasons": reasons, "samples": len(rows)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _build(args, rank, ws, log):
    from paper_1811_05731_b200.workloads import build_workload
    cache = args.cache_dir
    if ws > 1:
        import torch.distributed as dist
        if rank == 0:
            op, info = build_workload(args.config, cache_dir=cache, log=log)
        dist.barrier()
        if rank != 0:
            op, info = build_workload(args.config, cache_dir=cache, log=lambda *a: None)
        return op, info
    return build_workload(args.config, cache_dir=cache, log=log)


def _traffic(args):
    """DRAM bytes per launch of the dataflow kernel from the committed ncu
    capture of this workload (profiles/r01_traffic.json), or --traffic."""
    if args.traffic is not None:
        return args.traffic
    if args.nrhs != 1 or args.world > 1:
        return None
    try:
        t = json.loads((ROOT / "profiles" / "r01_traffic.json").read_text())
        return t[args.config]["bytes"]
    except (OSError, KeyError, ValueError):
        return None


L2_BYTES = 126 * 2**20


class DeviceTimer:
    """Device time of `fn` per step, CUDA events on `stream`.  With
    flush=True a buffer of twice the L2 is rewritten before every step,
    outside the timed interval, so no step finds the previous one's lines in
    L2."""

    def __init__(self, stream, flush=True):
        import torch
        self.torch = torch
        self.stream = stream
        self.buf = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device="cuda") if flush else None

    def run(self, fn, steps):
        torch = self.torch
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        with torch.cuda.stream(self.stream):
            if self.buf is None:
                ev[0][0].record(self.stream)
                for _ in range(steps):
                    fn()
                ev[0][1].record(self.stream)
                torch.cuda.synchronize()
                return ev[0][0].elapsed_time(ev[0][1]) / steps
            for k in range(steps):
                self.buf.fill_(k)
                ev[k][0].record(self.stream)
                fn()
                ev[k][1].record(self.stream)
            torch.cuda.synchronize()
        return sum(a.elapsed_time(b) for a, b in ev) / steps


def _config_block(args, n, op_bytes, extra=None):
    from paper_1811_05731_b200.workloads import WORKLOADS
    c = {"workload": f"{args.config}: {WORKLOADS[args.config]['desc']}", "n": n, "nrhs": args.nrhs,
         "h2_bytes": op_bytes, "parallelism": f"shard{args.world}" if args.world > 1 else "single",
         "l2": "flushed before every timed step (a 252 MB buffer rewritten outside the timed interval); "
               "the operator is also larger than the 126 MB L2" if args.l2_flush else
               "not flushed: the operator streamed per step is larger than the 126 MB L2"}
    if extra:
        c.update(extra)
    return c


def _cpu_port_single(op, x, seconds=10.0, max_reps=40):
    """Oracle port, one thread (threadpoolctl), bounded sample."""
    from oracle.h2_matvec_ref import h2_matvec_ref
    try:
        from threadpoolctl import threadpool_limits
        lim = threadpool_limits(1)
    except Exception:
        lim = None
    try:
        h2_matvec_ref(op, x)
        reps, t0 = 0, time.perf_counter()
        while reps < max_reps and (reps < 3 or time.perf_counter() - t0 < seconds):
            h2_matvec_ref(op, x)
            reps += 1
        dt = (time.perf_counter() - t0) / reps
    finally:
        if lim is not None:
            lim.unregister() if hasattr(lim, "unregister") else None
    return dt, reps


_POOL_OP = {}


def _pool_task(i):
    from oracle.h2_matvec_ref import h2_matvec_ref
    op = _POOL_OP["op"]
    x = np.random.default_rng(1234 + i).standard_normal(op.n)
    t = time.perf_counter()
    h2_matvec_ref(op, x)
    return time.perf_counter() - t


def run_reference(args):
    ws, rank, local = _dist()
    if ws > 1 and rank != 0:
        return 0  # rank 0 alone runs the CPU reference arm
    log = (lambda m: print(m, file=sys.stderr, flush=True))
    op, info = _build(args, 0, 1, log)
    import multiprocessing as mp
    cores = os.cpu_count() or 1
    _POOL_OP["op"] = op
    try:  # one BLAS thread per process; inherited by the forked workers
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        pool.map(_pool_task, range(min(args.warmup, cores) or 1))
        t0 = time.perf_counter()
        per = pool.map(_pool_task, range(args.steps), chunksize=1)
        wall = time.perf_counter() - t0
    value = args.steps * op.n * args.nrhs / wall
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": _config_block(args, op.n, op.storage_bytes()),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"{args.steps} full products of the workload, one per process on "
                                       f"{cores} processes (OPENBLAS_NUM_THREADS=1 each); mean single-product "
                                       f"latency {1e3 * float(np.mean(per)):.1f} ms"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_b200(args):
    import torch
    ws, rank, local = _dist()
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    log = (lambda m: print(m, file=sys.stderr, flush=True)) if rank == 0 else (lambda m: None)
    op, info = _build(args, rank, ws, log)
    from paper_1811_05731_b200.h2 import DeviceOperator, h2_matvec, h2_matmat, nccl_unique_id
    if ws > 1:
        obj = [nccl_unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(obj, src=0)
        dev = DeviceOperator(op, rank=rank, world_size=ws, nccl_unique_id=obj[0])
    else:
        dev = DeviceOperator(op)
    st = dev.stats()
    n, nrhs = op.n, args.nrhs
    from paper_1811_05731_b200.workloads import vector_for
    xh = vector_for(args.config, n, nrhs, seed=1234)
    x = torch.from_numpy(np.ascontiguousarray(xh)).cuda()
    y = torch.empty_like(x)
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    # parity spot-check of this very operator against the oracle (rank 0)
    parity = None
    if not args.profile:
        yg = dev.matvec(xh)   # full y on every rank (multi-GPU: rows assembled over NCCL)
    if rank == 0 and not args.profile:
        from oracle.h2_matvec_ref import h2_matvec_ref
        x0 = xh if nrhs == 1 else xh[:, 0]
        y0 = yg if nrhs == 1 else yg[:, 0]
        yr = h2_matvec_ref(op, x0)
        parity = float(np.linalg.norm(y0 - yr) / np.linalg.norm(yr))
    for _ in range(args.warmup):
        dev.matvec_dev(x.data_ptr(), y.data_ptr(), nrhs, sp)
    torch.cuda.synchronize()
    peaks, peak_kind = _peaks()
    timer = DeviceTimer(stream, flush=args.l2_flush)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ms = timer.run(lambda: dev.matvec_dev(x.data_ptr(), y.data_ptr(), nrhs, sp), args.steps)
    if ws > 1:
        torch.distributed.barrier()
    if ws > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    clocks = clk.summary(peaks.get("sm_max_mhz"))
    value = n * nrhs / (ms * 1e-3)          # one product of the whole operator per step
    b_alg = st["stream_bytes"] + 16 * n * nrhs
    achieved = b_alg / (ms * 1e-3) / 1e9   # aggregate over the GPUs
    # end to end through the public API with host buffers (pinned), rank-local
    e2e = None
    if not args.profile:
        xp = torch.from_numpy(np.ascontiguousarray(xh)).pin_memory().numpy()
        if ws > 1:
            call = lambda: dev.matvec(xp)    # the rank operator's host entry point
        else:
            call = (lambda: h2_matvec(op, xp)) if nrhs == 1 else (lambda: h2_matmat(op, xp))
        for _ in range(3):
            call()
        k = max(5, min(args.steps, 200))
        te = 0.0
        for i in range(k):
            if timer.buf is not None:  # same L2 treatment as the device-timed steps
                timer.buf.fill_(i)
                torch.cuda.synchronize()
            t0 = time.perf_counter()
            call()
            te += time.perf_counter() - t0
        te /= k
        if ws > 1:
            t = torch.tensor([te], device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            te = float(t.item())
        e2e = {"value": n * nrhs / te, "unit": UNIT, "h2d_bytes_per_step": 8 * n * nrhs,
               "d2h_bytes_per_step": 8 * n * nrhs, "ms_per_step": te * 1e3, "steps": k}
    cpu = None
    if rank == 0 and ws == 1 and not args.profile and not args.no_cpu_baseline:
        x0 = xh if nrhs == 1 else xh[:, 0]
        dt, reps = _cpu_port_single(op, x0)
        cpu = {"value": n / dt, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"{reps} single-vector products of the same operator, oracle/h2_matvec_ref.py "
                         f"(Python loop of numpy GEMVs like h2.py:186-244), 1 thread, "
                         f"{dt * 1e3:.1f} ms per product"}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "strong" if ws > 1 else "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": _config_block(args, n, op.storage_bytes(),
                                        {"build": {k: v for k, v in info.items() if k != "build_seconds"},
                                         "build_seconds": {k: round(v, 2) for k, v in
                                                           (info.get("build_seconds") or {}).items()},
                                         "work_items": st["ntasks"], "grid": st["grid"],
                                         "bytes_by_kind": st["bytes_by_kind"]}),
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"] * ws, "unit": "GB/s",
                             "frac": achieved / (peaks["hbm_gbs"] * ws), "traffic": _traffic(args),
                             "peak_kind": peak_kind, "aggregate_over_gpus": ws,
                             "algorithmic_bytes_per_launch": b_alg},
                "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": (2 if ws == 1 else 3) * args.steps, "clocks": clocks,
                "parity_rel_err_vs_oracle": parity}
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    dev.close()
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", default="config3")
    ap.add_argument("--nrhs", type=int, default=1)
    ap.add_argument("--cache-dir", default=os.environ.get("H2B_CACHE", "/tmp/h2b_cache"))
    ap.add_argument("--profile", action="store_true", help="skip parity/e2e/CPU legs (for ncu)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--l2-flush", action="store_true",
                    help="rewrite a 252 MB buffer before every timed step (default: K back-to-back "
                         "steps; the operator is larger than the L2 for configs 2-5)")
    ap.add_argument("--traffic", type=float, default=None,
                    help="ncu dram bytes per launch of the kernel (from profiles/), reported verbatim")
    args = ap.parse_args(argv)
    args.warmup = max(args.warmup, 3)
    args.world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.world == 1 and args.gpus != 1:
        print(f"note: --gpus {args.gpus} without torchrun runs one process on one GPU", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args)
    import __graft_entry__
    __graft_entry__.build()
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
