"""numpy interpreter of the libh2b execution plan — TEST INFRASTRUCTURE ONLY.

Executes the work-item queue exported by ``h2b_plan_view_get`` with exactly
the semantics the CUDA kernel implements (csrc/h2b.cu ``run_item``):

    out[0:m] = sum_j bias_slot_j[0:m] + A[0:m, 0:ncols] @ gather(segments)

where A is the column-major slice ``mat[data + c*ld + r]``.  Agreement of
this interpreter with the reference h2_matvec (h2.py:186-244) on CPU proves
the planner's layout, packing, splitting and dependency order before any GPU
runs; the GPU parity tests then only have to pin the kernel.
"""

from __future__ import annotations

import numpy as np

__all__ = ["run_plan", "run_phase", "run_ranks", "check_plan_invariants"]


def run_plan(plan: dict, x: np.ndarray, rng=None) -> np.ndarray:
    """Single-phase plan: y = M x (``rng``: random dependency-respecting order)."""
    x = np.asarray(x, dtype=np.float64)
    nrhs = 1 if x.ndim == 1 else x.shape[1]
    coef = np.full((max(1, plan["coef_len"]), nrhs), np.nan)
    Y = np.full((plan["n"], nrhs), np.nan)
    run_phase(plan, x, coef, Y, rng=rng)
    return Y[:, 0].copy() if x.ndim == 1 else Y


def run_ranks(rank_plans: list, x: np.ndarray) -> np.ndarray:
    """Emulate a multi-GPU product: phase 0 on every rank, the all-gather of
    the x^ exchange regions, phase 1 on every rank; each rank owns the rows
    of its leaves."""
    x = np.asarray(x, dtype=np.float64)
    nrhs = 1 if x.ndim == 1 else x.shape[1]
    W = len(rank_plans)
    coefs = [np.full((max(1, p["coef_len"]), nrhs), np.nan) for p in rank_plans]
    ys = [np.full((p["n"], nrhs), np.nan) for p in rank_plans]
    for r, p in enumerate(rank_plans):
        run_phase(p["phases"][0], x, coefs[r], ys[r])
    off, cnt = rank_plans[0]["exchange"]
    for r in range(W):
        region = coefs[r][off + r * cnt: off + (r + 1) * cnt].copy()
        for q in range(W):
            coefs[q][off + r * cnt: off + (r + 1) * cnt] = region
    for r, p in enumerate(rank_plans):
        run_phase(p["phases"][1], x, coefs[r], ys[r])
    Y = np.full_like(ys[0], np.nan)
    for r, p in enumerate(rank_plans):
        lo, hi = p["rank_lo_hi"][r]
        rows = p["perm"][lo:hi]
        assert not np.isnan(ys[r][rows]).any(), "rank left owned rows unwritten"
        Y[rows] = ys[r][rows]
    return Y[:, 0].copy() if x.ndim == 1 else Y


def run_phase(plan: dict, x: np.ndarray, coef: np.ndarray, Y: np.ndarray, rng=None) -> None:
    """Execute one phase.  Scheduled units are fused runs (t_mlen > 0 at
    their first item: items t .. t+L-1 run back to back, like one warp of
    the kernel).  In queue order by default; with ``rng`` in a random
    dependency-respecting order, as the dynamic scheduler may — inputs a
    unit does not declare would then read the NaN-initialised workspace."""
    nrhs = coef.shape[1]
    X = np.asarray(x, dtype=np.float64).reshape(plan["n"], nrhs)
    mat, perm = plan["mat"], plan["perm"]
    T = len(plan["t_m"])
    mlen = plan.get("t_mlen")
    if mlen is None:
        mlen = np.ones(T, np.int32)
    done = np.zeros(T, bool)
    t_seg0, t_dep0 = plan["t_seg0"], plan["t_dep0"]

    def execute(t):
        m, ld, nc = int(plan["t_m"][t]), int(plan["t_ld"][t]), int(plan["t_ncols"][t])
        src = []
        for s in range(t_seg0[t], t_seg0[t + 1]):
            k, a, w = int(plan["s_kind"][s]), int(plan["s_src"][s]), int(plan["s_ncols"][s])
            if k == 0:
                src.append(X[perm[a:a + w]])
            else:
                stride, ns = int(plan["s_stride"][s]), int(plan["s_nslots"][s])
                v = np.zeros((w, nrhs))
                for j in range(ns):
                    v = v + coef[a + j * stride: a + j * stride + w]
                src.append(v)
        xs = np.concatenate(src) if src else np.zeros((0, nrhs))
        assert xs.shape[0] == nc
        d0 = int(plan["t_data"][t])
        idx = d0 + np.arange(nc)[None, :] * ld + np.arange(m)[:, None]
        A = mat[idx] if nc else np.zeros((m, 0))
        acc = A @ xs
        b = int(plan["t_bias"][t])
        if b >= 0:
            st, ns = int(plan["t_bias_stride"][t]), int(plan["t_bias_nslots"][t])
            for j in range(ns):
                acc = acc + coef[b + j * st: b + j * st + m]
        o = int(plan["t_out"][t])
        if plan["t_kind"][t] == 4:
            Y[perm[o:o + m]] = acc
        else:
            coef[o:o + m] = acc
        done[t] = True

    def run_unit(t):
        deps = plan["deps"][t_dep0[t]:t_dep0[t + 1]]
        assert np.all(deps < t) and np.all(done[deps]), "dependency order violated"
        for j in range(int(mlen[t])):
            assert j == 0 or (mlen[t + j] == 0 and t_dep0[t + j] == t_dep0[t + j + 1])
            execute(t + j)

    units = [t for t in range(T) if mlen[t] > 0]
    assert sum(int(mlen[t]) for t in units) == T, "fused runs must tile the queue"
    # gated coupling rows: no listed dependencies, released once every
    # upward item (kinds 0, 1) of the phase has finished
    gated = set(int(g) for g in plan.get("gated", []))
    up_units = [t for t in units if plan["t_kind"][t] <= 1]
    assert len(up_units) == plan.get("n_up", len(up_units)) or not gated
    if rng is None:
        for t in units:
            if t in gated:
                assert all(done[u] for u in up_units), "gated item before the upward pass finished"
            run_unit(t)
        return
    remaining = {t: int(t_dep0[t + 1] - t_dep0[t]) for t in units}
    succ = {t: [] for t in units}
    for t in units:
        for d in plan["deps"][t_dep0[t]:t_dep0[t + 1]]:
            succ[int(d)].append(t)
    ready = [t for t in units if remaining[t] == 0 and t not in gated]
    up_left = len(up_units)
    if up_left == 0:
        ready.extend(sorted(gated))
    while ready:
        t = ready.pop(int(rng.integers(len(ready))))
        run_unit(t)
        if plan["t_kind"][t] <= 1:
            up_left -= 1
            if up_left == 0:
                ready.extend(sorted(gated))
        for s2 in succ[t]:
            remaining[s2] -= 1
            if remaining[s2] == 0:
                ready.append(s2)
    assert all(done), "some units never became ready"


def check_plan_invariants(plan: dict) -> None:
    """Structural invariants the kernel relies on."""
    T = len(plan["t_m"])
    assert np.all(plan["t_m"] >= 1) and np.all(plan["t_m"] <= 64)
    assert np.all(plan["t_ld"] >= plan["t_m"])
    for t in range(T):
        d = plan["deps"][plan["t_dep0"][t]:plan["t_dep0"][t + 1]]
        assert np.all(d < t)
        seg = slice(plan["t_seg0"][t], plan["t_seg0"][t + 1])
        assert plan["s_ncols"][seg].sum() == plan["t_ncols"][t]
    assert plan["mat"].size * 8 == sum(plan["stats"]["bytes_by_kind"].values())
    assert plan["mat"].size * 8 <= plan["stats"]["stream_bytes"] + plan["stats"]["extra_bytes"]
    # every y row written exactly once
    fin = np.flatnonzero(plan["t_kind"] == 4)
    rows = np.concatenate([plan["t_out"][t] + np.arange(plan["t_m"][t]) for t in fin])
    assert np.array_equal(np.sort(rows), np.arange(plan["n"]))
