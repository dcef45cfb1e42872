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

``--impl reference`` times the UNMODIFIED reference matvec
(``strayfield.hmatrix.h2.h2_matvec``, h2.py:186-244, imported from
baseline/_ref) on the host cores, one process per core, on an operator with
exactly the workload's structure (oracle/reference.py ``structure_twin``:
same tree, block partition and ranks -- hence the same GEMV shapes and
storage_bytes -- seeded entries), built on the host CPU only: this arm never
touches the GPU or loads a native library of this repo.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
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
    """DRAM bytes per product (every launch of a step, summed) from the
    committed ncu capture of this workload (profiles/r02_traffic.json, else
    the round-1 file), or --traffic."""
    if args.traffic is not None:
        return args.traffic
    if args.nrhs != 1 or args.world > 1:
        return None
    for name in ("r02_traffic.json", "r01_traffic.json"):
        try:
            t = json.loads((ROOT / "profiles" / name).read_text())
            return t[args.config]["bytes"]
        except (OSError, KeyError, ValueError):
            continue
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


def _config_block(args, n, op_bytes):
    """The workload description -- identical in both arms."""
    from paper_1811_05731_b200.workloads import WORKLOADS
    return {"workload": f"{args.config}: {WORKLOADS[args.config]['desc']}", "n": n, "nrhs": args.nrhs,
            "h2_bytes": op_bytes, "parallelism": f"shard{args.world}" if args.world > 1 else "single",
            "l2": "flushed before every timed step (a 252 MB buffer rewritten outside the timed interval); "
                  "the operator is also larger than the 126 MB L2" if args.l2_flush else
                  "not flushed: the operator streamed per step is larger than the 126 MB L2"}


def _peak_rss_gb():
    import resource
    return resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6


def _loaded_native():
    """In-tree shared objects mapped into this process."""
    try:
        maps = Path("/proc/self/maps").read_text()
    except OSError:
        return None
    return sorted({ln.split()[-1] for ln in maps.splitlines()
                   if ln.endswith(".so") and str(ROOT) in ln})


def _cpu_reference_single(op, x, seconds=10.0, max_reps=40):
    """The unmodified reference h2_matvec (baseline/_ref) on the same
    operator, one BLAS thread, bounded sample; the oracle port when the
    reference is not vendored."""
    try:
        from oracle.reference import available, reference_h2_matvec, to_reference
        if not available():
            raise ImportError
        fn, target, kind = reference_h2_matvec(), to_reference(op), "reference"
    except ImportError:
        from oracle.h2_matvec_ref import h2_matvec_ref
        fn, target, kind = h2_matvec_ref, op, "port"
    try:
        from threadpoolctl import threadpool_limits
        lim = threadpool_limits(1)
    except Exception:
        lim = None
    try:
        fn(target, x)
        reps, t0 = 0, time.perf_counter()
        while reps < max_reps and (reps < 3 or time.perf_counter() - t0 < seconds):
            fn(target, x)
            reps += 1
        dt = (time.perf_counter() - t0) / reps
    finally:
        if lim is not None:
            lim.restore_original_limits()
    return dt, reps, kind


def _ref_worker(op, n_products, nrhs, barrier, q, seed):
    """One reference process: warm-up product, then n_products timed ones
    (each product of a multi-RHS step is nrhs single-vector calls: the
    reference has no multi-RHS entry point)."""
    from oracle.reference import reference_h2_matvec
    fn = reference_h2_matvec()
    x = np.random.default_rng(seed).standard_normal(op.n)
    fn(op, x)
    barrier.wait()
    t0 = time.perf_counter()
    for _ in range(n_products * nrhs):
        fn(op, x)
    q.put((t0, time.perf_counter()))


def run_reference(args):
    ws, rank, local = _dist()
    if ws > 1 and rank != 0:
        return 0  # rank 0 alone runs the CPU reference arm
    log = (lambda m: print(m, file=sys.stderr, flush=True))
    import multiprocessing as mp
    from oracle.reference import available, rank_fixture_path, structure_twin, to_reference
    name = "config3" if args.config == "config4" else args.config
    why = None
    if not available():
        why = "baseline/_ref is not vendored (tools/vendor_reference.sh)"
    elif not rank_fixture_path(name).exists():
        why = f"no structure fixture {rank_fixture_path(name).name} for {args.config}"
    if why:
        print(json.dumps({"impl": "reference", "unavailable": why}), flush=True)
        return 0
    twin, info = structure_twin(name, log=log)
    op = to_reference(twin)
    cores = os.cpu_count() or 1
    try:  # one BLAS thread per process; inherited by the forked workers
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass
    per_proc = max(1, -(-args.steps // cores))   # ceil: every core runs the same count
    ctx = mp.get_context("fork")
    barrier, q = ctx.Barrier(cores), ctx.Queue()
    procs = [ctx.Process(target=_ref_worker, args=(op, per_proc, args.nrhs, barrier, q, 1234 + i))
             for i in range(cores)]
    for p_ in procs:
        p_.start()
    spans = [q.get() for _ in procs]
    for p_ in procs:
        p_.join()
    wall = max(b for _, b in spans) - min(a for a, _ in spans)
    total = cores * per_proc
    value = total * op.n * args.nrhs / wall
    lat = float(np.mean([(b - a) / (per_proc * args.nrhs) for a, b in spans]))
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / total,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": _config_block(args, op.n, twin.storage_bytes()),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                             "sample": f"{total} products ({per_proc} per process on {cores} processes, "
                                       f"OPENBLAS_NUM_THREADS=1 each, after one warm-up product each) of the "
                                       f"unmodified strayfield.hmatrix.h2.h2_matvec from baseline/_ref on an "
                                       f"operator with the workload's exact structure (tree, blocks, ranks: "
                                       f"{twin.storage_bytes()} bytes) and seeded entries; mean single-product "
                                       f"latency {1e3 * lat:.1f} ms"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "build": {"twin_seconds": round(info["build_seconds"], 1)},
            "native_so_loaded": _loaded_native(), "host_peak_rss_gb": round(_peak_rss_gb(), 1)}
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
    from paper_1811_05731_b200.h2 import DeviceOperator, device_operator, h2_matvec, h2_matmat, nccl_unique_id
    if ws > 1:
        obj = [nccl_unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(obj, src=0)
        dev = DeviceOperator(op, rank=rank, world_size=ws, nccl_unique_id=obj[0])
    else:
        dev = device_operator(op)   # the one h2_matvec(op, x) uses: one device copy
    log(f"[bench] device operator ready [host peak rss {_peak_rss_gb():.1f} GB]")
    st = dev.stats()
    n, nrhs = op.n, args.nrhs
    from paper_1811_05731_b200.workloads import vector_for, z_over_3
    xh = vector_for(args.config, n, nrhs, seed=1234)
    x = torch.from_numpy(np.ascontiguousarray(xh)).cuda()
    y = torch.empty_like(x)
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    # parity of this very operator against the oracle (rank 0): every column
    # of the seeded N(0,1) input and, where the node coordinates are known,
    # u1 = z/3 (BASELINE configs 1 and 5)
    parity = None
    if not args.profile:
        vecs = {"randn": xh}
        if info.get("coords") is not None and nrhs == 1:
            vecs["z_over_3"] = z_over_3(info["coords"])
        ys = {k: dev.matvec(v) for k, v in vecs.items()}   # multi-GPU: rows assembled over NCCL
    if rank == 0 and not args.profile:
        from oracle.h2_matvec_ref import h2_matvec_ref
        parity = {}
        for k, v in vecs.items():
            cols = [v] if v.ndim == 1 else [v[:, j] for j in range(v.shape[1])]
            ycols = [ys[k]] if v.ndim == 1 else [ys[k][:, j] for j in range(v.shape[1])]
            errs = []
            for xc, yc in zip(cols, ycols):
                yr = h2_matvec_ref(op, np.ascontiguousarray(xc))
                errs.append(float(np.linalg.norm(yc - yr) / np.linalg.norm(yr)))
            parity[k] = max(errs)
            log(f"[bench] parity {k}: {parity[k]:.2e} over {len(errs)} column(s)")
    # compression error of the built operator itself (rank 0): sampled rows of
    # the exact collocation matrix (GPU collocation kernel) times the seeded
    # input against the same rows of the H² product.  By default when the
    # operator was built in this run (its surface is at hand).
    op_check = None
    rows_wanted = args.check_rows if args.check_rows is not None else (32 if info.get("surface") is not None else 0)
    if rank == 0 and not args.profile and rows_wanted > 0:
        from paper_1811_05731_b200.workloads import exact_rows, surface_for
        surf = info.get("surface") or surface_for(args.config)
        nodes = np.sort(np.random.default_rng(99).choice(n, size=min(rows_wanted, n), replace=False))
        rows = exact_rows(surf, nodes)
        x0 = xh if xh.ndim == 1 else xh[:, 0]
        y0 = ys["randn"] if xh.ndim == 1 else ys["randn"][:, 0]
        exact = rows @ x0
        scale = float(np.linalg.norm(y0) / np.sqrt(n))   # rms of y
        err = np.abs(y0[nodes] - exact) / scale
        rsum = rows.sum(axis=1)   # (M 1)_i: the same constant for every node of a closed surface
        op_check = {"rows": int(nodes.size), "max_err_over_rms_y": float(err.max()),
                    "rms_err_over_rms_y": float(np.sqrt(np.mean(err ** 2))),
                    "exact_row_sum_mean": float(rsum.mean()), "exact_row_sum_spread": float(np.ptp(rsum)),
                    "note": "exact rows of M = K + D by the collocation kernel (bem.py:221-235) times the seeded "
                            "input vs the same rows of the H² product; the operator was compressed with "
                            "eps 1e-5 / eps_rec 2e-4"}
        log(f"[bench] operator check: {nodes.size} exact rows, max err {err.max():.2e}, rms {op_check['rms_err_over_rms_y']:.2e} (of rms y)")
        del rows
    info.pop("surface", None)
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
    # end to end through the public API with host buffers: the pageable
    # numpy arrays the real callers pass (apply_operator, compute_demag) --
    # the headline -- and, beside it, pinned host arrays
    e2e = None
    e2e_pinned = None
    if not args.profile:
        def e2e_time(xin):
            if ws > 1:
                call = lambda: dev.matvec(xin)    # the rank operator's host entry point
            else:
                call = (lambda: h2_matvec(op, xin)) if nrhs == 1 else (lambda: h2_matmat(op, xin))
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
            return {"value": n * nrhs / te, "unit": UNIT, "h2d_bytes_per_step": 8 * n * nrhs,
                    "d2h_bytes_per_step": 8 * n * nrhs, "ms_per_step": te * 1e3, "steps": k}
        e2e = e2e_time(np.ascontiguousarray(xh))
        e2e["host_input"] = "pageable numpy array (as apply_operator / compute_demag pass it)"
        e2e_pinned = e2e_time(torch.from_numpy(np.ascontiguousarray(xh)).pin_memory().numpy())
        e2e_pinned["host_input"] = "pinned"
    # per-launch device times (CUDA events around every launch, on the
    # launching stream): the dominant kernel's own roofline beside the whole
    # product's
    kernels = None
    dominant = None
    if ws == 1:
        kernels = dev.launch_times(x.data_ptr(), y.data_ptr(), nrhs, max(3, min(20, args.steps)), sp)
        xy = 16 * n * nrhs
        for kd in kernels:
            kd["GB/s"] = round(kd["bytes"] / (kd["ms"] * 1e-3) / 1e9, 1) if kd["ms"] > 0 and kd["bytes"] else None
        dominant = max(kernels, key=lambda kd: kd["ms"])
        tot = sum(kd["ms"] for kd in kernels)
        dominant = {"kernel": dominant["kernel"], "ms": dominant["ms"], "share_of_step": dominant["ms"] / tot,
                    "algorithmic_bytes": dominant["bytes"],
                    "achieved": dominant["bytes"] / (dominant["ms"] * 1e-3) / 1e9,
                    "frac": dominant["bytes"] / (dominant["ms"] * 1e-3) / 1e9 / peaks["hbm_gbs"]}
    nlaunch = len(dev.launches(nrhs)) + (1 if ws > 1 else 0)   # multi-GPU: + the x^ all-gather (NCCL)
    cpu = None
    if rank == 0 and ws == 1 and not args.profile and not args.no_cpu_baseline:
        x0 = xh if nrhs == 1 else np.ascontiguousarray(xh[:, 0])
        dt, reps, kind = _cpu_reference_single(op, x0)
        what = ("the unmodified strayfield.hmatrix.h2.h2_matvec (baseline/_ref, h2.py:186-244)" if kind == "reference"
                else "oracle/h2_matvec_ref.py (restatement of h2.py:186-244)")
        cpu = {"value": n / dt, "unit": UNIT, "cores": 1, "kind": kind,
               "sample": f"{reps} single-vector products of the same operator, {what}, 1 thread, "
                         f"{dt * 1e3:.1f} ms per product"}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "strong" if ws > 1 else "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": _config_block(args, n, op.storage_bytes()),
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"] * ws, "unit": "GB/s",
                             "frac": achieved / (peaks["hbm_gbs"] * ws), "traffic": _traffic(args),
                             "peak_kind": peak_kind, "aggregate_over_gpus": ws,
                             "algorithmic_bytes_per_launch": b_alg,
                             "scope": "the whole product (every launch of a step)",
                             "dominant_kernel": dominant, "kernels": kernels},
                "cpu_baseline": cpu, "e2e": e2e, "e2e_pinned": e2e_pinned,
                "gpu_launches": nlaunch * args.steps, "clocks": clocks,
                "parity_rel_err_vs_oracle": max(parity.values()) if parity else None,
                "parity": parity,
                "operator_check": op_check,
                "build": {**{k: v for k, v in info.items() if k not in ("build_seconds", "coords")},
                          "seconds": {k: round(v, 2) for k, v in (info.get("build_seconds") or {}).items()}},
                "plan": {"work_items": st["ntasks"], "grid": st["grid"], "bytes_by_kind": st["bytes_by_kind"]},
                "host_peak_rss_gb": round(_peak_rss_gb(), 1)}
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
    ap.add_argument("--check-rows", type=int, default=None,
                    help="exact collocation rows to check the built operator against (default: 32 when the "
                         "operator was built in this run, else 0)")
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
