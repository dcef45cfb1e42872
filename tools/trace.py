"""Per-work-item timeline of one H² product (diagnostics).

    python tools/trace.py --config config2 [--ablate far|near] [--opts '{}']

Prints per-kind item statistics and the critical path: walking back from
the last item to finish, each step goes to the predecessor that finished
last, with the gap between that predecessor's end and the item's start
(scheduling latency) and the item's own duration."""

import argparse
import ctypes as C
import dataclasses
import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

KINDS = ("up_leaf", "up_node", "down", "near", "final")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="config2")
    ap.add_argument("--cache-dir", default="/tmp/h2b_cache")
    ap.add_argument("--ablate", default="")
    ap.add_argument("--opts", default="{}")
    ap.add_argument("--save", default="")
    ap.add_argument("--nrhs", type=int, default=1)
    ap.add_argument("--phase", type=int, default=-1,
                    help="launch of the plan to trace (staged plans: 0 up sweep, 1 dataflow, 2 down sweep); "
                         "default: the first dataflow launch")
    a = ap.parse_args()
    import torch
    import __graft_entry__
    __graft_entry__.build()
    from paper_1811_05731_b200 import _native as nat
    from paper_1811_05731_b200.h2 import DeviceOperator, plan_view
    from paper_1811_05731_b200.workloads import build_workload, vector_for
    op, _ = build_workload(a.config, cache_dir=a.cache_dir, log=lambda m: print(m, file=sys.stderr))
    if a.ablate == "far":
        op = dataclasses.replace(op, near=[])
    elif a.ablate == "near":
        op = dataclasses.replace(op, coupling=[])
    elif a.ablate == "chain":  # bases and transfers only: the bare tree chain
        op = dataclasses.replace(op, near=[], coupling=[])
    opts = json.loads(a.opts)
    split = a.nrhs >= 8 and os.environ.get("H2B_NEAR_SPLIT", "1") != "0"
    if split:   # trace the dataflow part of the split multi-RHS product
        os.environ["H2B_TRACE_SPLIT"] = "1"
        # the split product's dataflow part is the last launch of the view;
        # 8/16 right-hand sides may run the classic (unstaged) split plan:
        # the candidate whose size the library accepts is the one traced
        cands = []
        for extra in (4, 4 | 2048):
            pv = plan_view(op, **dict(opts, plan_flags=opts.get("plan_flags", 0) | extra))
            ph = pv["phases"][-1]
            ph["stats"] = pv["stats"]
            cands.append(ph)
        plan = cands[0]
    else:
        pv = plan_view(op, **opts)
        k = a.phase if a.phase >= 0 else [ph["mode"] for ph in pv["phases"]].index(0)
        os.environ["H2B_TRACE_PHASE"] = str(k)
        plan = pv["phases"][k]
        plan["stats"] = pv["stats"]
        print(f"launches: {[(ph['mode'], len(ph['t_m'])) for ph in pv['phases']]}, tracing launch {k}")
    dev = DeviceOperator(op, **opts)
    lib = nat.lib()
    lib.h2b_trace_enable.argtypes = [C.c_void_p, C.c_int]
    lib.h2b_trace_read.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
    nrhs = a.nrhs
    x = torch.from_numpy(np.ascontiguousarray(vector_for(a.config, op.n, nrhs))).cuda()
    y = torch.empty_like(x)
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(5):
        dev.matvec_dev(x.data_ptr(), y.data_ptr(), nrhs, s)
    nat.check(lib.h2b_trace_enable(dev._h, 1))
    for _ in range(3):
        dev.matvec_dev(x.data_ptr(), y.data_ptr(), nrhs, s)
    torch.cuda.synchronize()
    if split:
        for ph in cands:
            tr = np.zeros((ph["t_m"].size, 8), np.uint64)
            if lib.h2b_trace_read(dev._h, tr.ctypes.data, ph["t_m"].size) == 0:
                plan = ph
                break
    T = plan["t_m"].size
    tr = np.zeros((T, 8), np.uint64)
    nat.check(lib.h2b_trace_read(dev._h, tr.ctypes.data, T))
    # the resident sweep kernel ran only if the units fit shared memory at this nrhs (h2b_stats.resident_mask)
    res_ran = bool(dev.stats().get("resident_mask", 0) & nrhs)
    if plan.get("mode", 0) == 1 and plan.get("resident") and res_ran and os.environ.get("H2B_SWEEP_RESIDENT", "1") != "0":
        # resident sweep: one record per unit, in the slots of its first item:
        # start, end, waves | cta, copies issued, copies landed, end of wave 0, 1, last but one
        first = plan["wave0"][plan["unit0"][:-1]]
        r = tr[first].astype(np.int64)
        ok = r[:, 1] > 0
        r = r[ok]
        t0 = r[:, 0].min()
        print(f"resident sweep: {ok.sum()} units of {len(first)}, span {(r[:, 1].max() - t0) / 1e3:.1f} us, "
              f"first start {0.0:.1f}, last start {(r[:, 0].max() - t0) / 1e3:.1f} us")
        names = ("issue", "land", "wave0", "wave1", "..last-1", "last")
        cols = [(0, 3), (3, 4), (4, 5), (5, 6), (6, 7), (7, 1)]
        print("  per unit us: " + " ".join(f"{n} {(r[:, b] - r[:, a]).clip(0).mean() / 1e3:5.2f}" for n, (a, b) in zip(names, cols))
              + f"  total {(r[:, 1] - r[:, 0]).mean() / 1e3:5.2f}  waves {np.mean(r[:, 2] >> 32):.1f}")
        R = plan["u_range"]
        print(f"  per unit KB: matrices {R[:, 1].mean() * 8 / 1e3:.1f} coef {R[:, 3].mean() * 8 / 1e3:.1f} "
              f"partials {R[:, 5].mean() * 8 / 1e3:.1f} items {np.diff(plan['wave0'][plan['unit0']]).mean():.1f}")
        return
    # one record per scheduled unit (the first item of a fused run)
    unit = tr[:, 1] > 0
    start = tr[:, 0].astype(np.int64)
    end = tr[:, 1].astype(np.int64)
    t0 = start[unit].min()
    start[~unit] = t0
    end[~unit] = t0
    start -= t0
    end -= t0
    kind = plan["t_kind"]
    dur = end - start
    # stages: descriptor fetch, gather (+ staged matrix), compute, successors
    ts = tr[:, 0].astype(np.int64)
    td, tg, tr_ = (tr[:, j].astype(np.int64) for j in (5, 6, 4))
    tg = np.where(tg > 0, tg, td)
    t_desc, t_gath, t_comp = td - ts, tg - td, tr_ - tg
    t_succ = tr[:, 1].astype(np.int64) - tr_
    nbytes = 8 * plan["t_m"].astype(np.int64) * plan["t_ncols"]
    print(f"items {T}, span {end.max() / 1e3:.1f} us, bytes {nbytes.sum() / 1e6:.1f} MB")
    if plan.get("mode", 0) == 1:
        # sweeps record more stages: descriptors and prefetch issue, segment
        # table, gather, wait for the staged matrix, multiply, store
        seg, gat = tr[:, 3].astype(np.int64), tr[:, 7].astype(np.int64)
        for k in range(5):
            sel = (kind == k) & unit & (seg > 0)
            if sel.any():
                parts = [td - ts, seg - td, gat - seg, tg - gat, tr_ - tg, tr[:, 1].astype(np.int64) - tr_]
                print(f"  {KINDS[k]:8s} stages us: " + " ".join(
                    f"{nm} {v[sel].mean() / 1e3:5.2f}" for nm, v in zip(("desc", "segtab", "gather", "wait", "fma", "store"), parts)))
    mlen = plan.get("t_mlen", np.ones(T, np.int32))
    print(f"units {int(unit.sum())}, fused runs {int((mlen > 1).sum())} (mean length "
          f"{mlen[mlen > 1].mean() if (mlen > 1).any() else 0:.1f})")
    for k in range(5):
        sel = (kind == k) & unit
        if sel.any():
            print(f"  {KINDS[k]:8s} n={sel.sum():6d} dur mean {dur[sel].mean() / 1e3:6.2f} us "
                  f"(desc {t_desc[sel].mean() / 1e3:5.2f} gath {t_gath[sel].mean() / 1e3:5.2f} comp {t_comp[sel].mean() / 1e3:5.2f} succ {t_succ[sel].mean() / 1e3:5.2f})  "
                  f"p90 {np.percentile(dur[sel], 90) / 1e3:6.2f}  start [{start[sel].min() / 1e3:7.1f}, "
                  f"{start[sel].max() / 1e3:7.1f}]  end max {end[sel].max() / 1e3:7.1f} us  "
                  f"MB {nbytes[sel].sum() / 1e6:7.1f}")
    # critical path
    dep0, deps = plan["t_dep0"], plan["deps"]
    cur = int(np.argmax(end))
    path = []
    while True:
        d = deps[dep0[cur]:dep0[cur + 1]]
        if d.size == 0:
            path.append((cur, None))
            break
        last = int(d[np.argmax(end[d])])
        path.append((cur, last))
        cur = last
    print(f"critical path: {len(path)} items")
    for it, pred in path[::-1]:
        gap = (start[it] - end[pred]) / 1e3 if pred is not None else start[it] / 1e3
        print(f"  {KINDS[kind[it]]:8s} L={mlen[it]:2d} m={plan['t_m'][it]:3d} ncols={plan['t_ncols'][it]:4d} "
              f"ndeps={dep0[it + 1] - dep0[it]:3d} start {start[it] / 1e3:7.1f} dur {dur[it] / 1e3:5.2f} "
              f"[desc {t_desc[it] / 1e3:5.2f} gath {t_gath[it] / 1e3:5.2f} comp {t_comp[it] / 1e3:5.2f} succ {t_succ[it] / 1e3:5.2f}] "
              f"gap {gap:5.2f} us sm={int(tr[it, 2]) >> 32} cont={int(tr[it, 3]) > 0}")
    # warps busy over time
    bins = np.linspace(0, end.max(), 21)
    busy = [(np.minimum(end, b1) - np.maximum(start, b0)).clip(0).sum() / (b1 - b0) for b0, b1 in zip(bins, bins[1:])]
    print("avg busy warps per 5% of span:", " ".join(f"{b:.0f}" for b in busy))
    # where each kind's bytes stream: MB per 5% of span (pro rata over each
    # item's interval); down items split into transfer pieces (a down
    # predecessor) and coupling pieces
    dk = np.zeros(T, bool)
    for it in np.nonzero(kind == 2)[0]:
        d = deps[dep0[it]:dep0[it + 1]]
        dk[it] = bool(d.size) and bool((kind[d] == 2).any())
    groups = [("up", (kind <= 1)), ("down-xfer", (kind == 2) & dk), ("down-coupl", (kind == 2) & ~dk),
              ("near", kind == 3), ("final", kind == 4)]
    span = np.maximum(end - start, 1)
    for name, sel in groups:
        sel = sel & unit
        row = [(nbytes[sel] * (np.minimum(end[sel], b1) - np.maximum(start[sel], b0)).clip(0) / span[sel]).sum() / 1e6
               for b0, b1 in zip(bins, bins[1:])]
        print(f"  MB/5% {name:10s}", " ".join(f"{r:6.0f}" for r in row))
    if a.save:
        np.savez_compressed(a.save, start=start, end=end, kind=kind, tr=tr, t_m=plan["t_m"],
                            t_ncols=plan["t_ncols"], dep0=dep0, deps=deps, t_out=plan["t_out"],
                            t_bias=plan["t_bias"], t_bias_nslots=plan["t_bias_nslots"])


if __name__ == "__main__":
    main()
