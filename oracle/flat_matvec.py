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

__all__ = ["run_plan", "run_phase", "run_group", "run_ranks", "check_plan_invariants", "launches"]


def launches(plan: dict, group=None, split: bool = False) -> list:
    """The launches of a plan in order (``h2b_plan_view.mode/group/split``):
    those of the plain product, or of the split multi-RHS product."""
    return [ph for ph in plan.get("phases", [plan])
            if bool(ph.get("split", 0)) == split and (group is None or ph.get("group", 0) == group)]


def run_group(plan: dict, group, x, coef, Y, rng=None, split: bool = False) -> None:
    """Every launch of one group (0: before the x^ exchange, 1: after), in order."""
    for ph in launches(plan, group, split):
        run_phase(ph, x, coef, Y, rng=rng)


def run_plan(plan: dict, x: np.ndarray, rng=None, split: bool = False) -> np.ndarray:
    """Single-GPU plan: y = M x, launch after launch (``rng``: random
    dependency-respecting order inside every launch; ``split``: the launches
    of the split multi-RHS product)."""
    x = np.asarray(x, dtype=np.float64)
    nrhs = 1 if x.ndim == 1 else x.shape[1]
    coef = np.full((max(1, plan["coef_len"]), nrhs), np.nan)
    Y = np.full((plan["n"], nrhs), np.nan)
    run_group(plan, None, x, coef, Y, rng=rng, split=split)
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
        run_group(p, 0, x, coefs[r], ys[r])
    off, cnt = rank_plans[0]["exchange"]
    for r in range(W):
        region = coefs[r][off + r * cnt: off + (r + 1) * cnt].copy()
        for q in range(W):
            coefs[q][off + r * cnt: off + (r + 1) * cnt] = region
    for r, p in enumerate(rank_plans):
        run_group(p, 1, x, coefs[r], ys[r])
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
    if plan.get("mode", 0) == 1:
        _run_sweep(plan, units, mlen, execute, coef, rng)
        assert all(done)
        return
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


def _run_sweep(plan, units, mlen, execute, coef, rng) -> None:
    """A sweep launch (csrc/h2b.cu h2b_sweep_kernel): every unit is run by
    one CTA, wave after wave with a block barrier between waves; the items
    of a wave run concurrently on the CTA's warps, so none may read what
    another of the same wave writes -- each wave is executed against a
    snapshot of the workspace taken at its start (and in a random order
    with ``rng``); units run in any order."""
    unit0, wave0 = plan["unit0"], plan["wave0"]
    assert len(unit0) - 1 == len(units) and wave0[-1] == len(plan["t_m"]) and len(plan["deps"]) == 0
    order = list(range(len(units)))
    if rng is not None:
        rng.shuffle(order)
    for u in order:
        assert wave0[unit0[u]] == units[u] and wave0[unit0[u + 1]] == units[u] + int(mlen[units[u]])
        for w in range(unit0[u], unit0[u + 1]):
            items = list(range(wave0[w], wave0[w + 1]))
            assert items, "empty wave"
            if rng is not None:
                rng.shuffle(items)
            before = coef.copy()
            written = np.zeros(coef.shape[0], bool)
            for t in items:
                # inputs as they were when the wave started
                mine = coef.copy()
                coef[:] = before
                execute(t)
                o, m = int(plan["t_out"][t]), int(plan["t_m"][t])
                if plan["t_kind"][t] != 4:
                    mine[o:o + m] = coef[o:o + m]
                    assert not written[o:o + m].any(), "two items of a wave write one slot"
                    written[o:o + m] = True
                coef[:] = mine


def check_plan_invariants(plan: dict) -> None:
    """Structural invariants the kernels rely on (every launch of the plain
    product of a single-GPU plan)."""
    rows = []
    for ph in launches(plan):
        T = len(ph["t_m"])
        assert np.all(ph["t_m"] >= 1) and np.all(ph["t_m"] <= 64)
        assert np.all(ph["t_ld"] >= ph["t_m"])
        for t in range(T):
            d = ph["deps"][ph["t_dep0"][t]:ph["t_dep0"][t + 1]]
            assert np.all(d < t)
            seg = slice(ph["t_seg0"][t], ph["t_seg0"][t + 1])
            assert ph["s_ncols"][seg].sum() == ph["t_ncols"][t]
        fin = np.flatnonzero(ph["t_kind"] == 4)
        rows += [ph["t_out"][t] + np.arange(ph["t_m"][t]) for t in fin]
    assert plan["mat"].size * 8 == sum(plan["stats"]["bytes_by_kind"].values())
    assert plan["mat"].size * 8 <= plan["stats"]["stream_bytes"] + plan["stats"]["extra_bytes"]
    # every y row written exactly once
    assert np.array_equal(np.sort(np.concatenate(rows)), np.arange(plan["n"]))
