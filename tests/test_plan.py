"""Host-side layout tests (no GPU): the C++ planner's work-item queue,
executed by the numpy interpreter in oracle/flat_matvec.py, must reproduce
the reference product; the C ABI must load and export every declared
symbol and reject malformed operators with the reference's error types."""

import ctypes
import dataclasses
import re

import numpy as np
import pytest

from conftest import ROOT, load_golden, rel
from oracle.flat_matvec import check_plan_invariants, run_plan
from oracle.h2_matvec_ref import h2_matvec_ref
from paper_1811_05731_b200 import _native as nat
from paper_1811_05731_b200.h2 import PLAN_NO_STAGED, plan_view
from synth import random_h2


def test_abi_exports_every_declared_symbol():
    header = (ROOT / "include" / "h2b.h").read_text()
    names = re.findall(r"^\s*(?:int|void|int64_t|const char\*)\s+\**(h2b_\w+)\s*\(", header, re.M)
    assert len(names) >= 12
    lib = ctypes.CDLL(str(nat.LIB_PATH))
    for nm in names:
        assert hasattr(lib, nm), nm
    assert nat.lib().h2b_abi_version() == 4


@pytest.mark.parametrize("task_bytes", [0, 4096, 512])
def test_plan_matches_reference(golden, task_bytes):
    name, op, ex = golden
    P = plan_view(op, task_bytes=task_bytes)
    check_plan_invariants(P)
    assert P["stats"]["stream_bytes"] == int(ex["storage_bytes"])
    Y = run_plan(P, ex["X"])
    for i in range(ex["X"].shape[1]):
        assert rel(Y[:, i], ex["y_full"][:, i]) <= 1e-14, (name, i)


def test_plan_far_and_near_ablations(golden):
    name, op, ex = golden
    x = ex["X"][:, 0]
    for abl, key in ((dataclasses.replace(op, coupling=[]), "y_near"),
                     (dataclasses.replace(op, near=[]), "y_far")):
        y = run_plan(plan_view(abl), x)
        ref = ex[key][:, 0]
        assert rel(y, ref) <= 1e-13, (name, key)


@pytest.mark.parametrize("opts", [dict(far_task_bytes=8192), dict(sched_flags=2), dict(sched_flags=2, far_task_bytes=8192),
                                  dict(far_task_bytes=8192, task_bytes=131072), dict(far_task_bytes=8192, task_bytes=262144)])
def test_plan_streaming_options(golden, opts):
    """The planning side of the streaming defaults (8 KB far-field pieces,
    finals in the slack queue) keeps the product exact."""
    name, op, ex = golden
    P = plan_view(op, **opts)
    check_plan_invariants(P)
    assert rel(run_plan(P, ex["X"][:, 0]), ex["y_full"][:, 0]) <= 1e-14


def test_plan_small_items(golden):
    name, op, ex = golden
    P = plan_view(op, task_bytes=256)
    check_plan_invariants(P)
    assert rel(run_plan(P, ex["X"][:, 0]), ex["y_full"][:, 0]) <= 1e-14


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("task_bytes", [0, 700])
def test_plan_random_structures(seed, task_bytes):
    op = random_h2(seed)
    P = plan_view(op, task_bytes=task_bytes)
    check_plan_invariants(P)
    assert P["stats"]["stream_bytes"] == op.storage_bytes()
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((op.n, 2))
    Y = run_plan(P, X)
    for i in range(2):
        assert rel(Y[:, i], h2_matvec_ref(op, X[:, i])) <= 1e-13


def test_plan_multi_rhs_layout():
    op, ex = load_golden("sphere3_l32_eta2_o4")
    X = ex["X"][:, :4]
    Y = run_plan(plan_view(op), X)
    for i in range(4):
        assert rel(Y[:, i], ex["y_full"][:, i]) <= 1e-14


def test_invalid_operators_rejected():
    op, _ = load_golden("sphere3_l32_eta2_o4")
    r, s, m = op.near[0]
    bad = dataclasses.replace(op, near=[(r, s, m[:, :-1])] + op.near[1:])
    with pytest.raises(ValueError):
        plan_view(bad)
    bad_perm = dataclasses.replace(op, tree=dataclasses.replace(op.tree, perm=np.zeros(op.n, np.int64)))
    with pytest.raises(ValueError, match="permutation"):
        plan_view(bad_perm)


def test_stats_kinds_cover_all_bytes(golden):
    name, op, ex = golden
    st = plan_view(op)["stats"]
    # the level-skipping chain (default below 4 GiB) adds its transfer
    # products and no longer reads the transfers of the skipped "own" levels
    assert sum(st["bytes_by_kind"].values()) == st["pool_bytes"] <= st["stream_bytes"] + st["extra_bytes"]
    assert st["stream_bytes"] == op.storage_bytes()
    st0 = plan_view(op, plan_flags=2)["stats"]   # H2B_PLAN_NO_SKIP: exactly storage_bytes
    assert sum(st0["bytes_by_kind"].values()) == op.storage_bytes() and st0["extra_bytes"] == 0
    assert st["tasks_by_kind"]["final"] == sum(1 for c in op.tree.clusters if c.is_leaf)


@pytest.mark.parametrize("band_depth", [1, 2, 3, 5])
def test_fused_runs_any_order(golden, band_depth):
    """Fused runs of the far-field chain: every unit declares
    all its external inputs, so any dependency-respecting order of the units
    (as the kernel's dynamic scheduler may pick) reproduces the reference."""
    name, op, ex = golden
    P = plan_view(op, band_depth=band_depth, far_task_bytes=1024, plan_flags=PLAN_NO_STAGED)
    check_plan_invariants(P)
    mlen = P["t_mlen"]
    if band_depth == 1:
        assert np.all(mlen == 1)
    elif name.startswith("config1"):  # depth-6 tree: the chain is fused
        assert mlen.max() > 1
    for seed in range(2):
        y = run_plan(P, ex["X"][:, 0], rng=np.random.default_rng(seed))
        assert rel(y, ex["y_full"][:, 0]) <= 1e-14, (name, band_depth, seed)


@pytest.mark.parametrize("seed", range(3))
def test_fused_runs_random_structures(seed):
    op = random_h2(seed)
    for bd in (2, 4):
        P = plan_view(op, band_depth=bd, task_bytes=700, plan_flags=PLAN_NO_STAGED)
        x = np.random.default_rng(seed).standard_normal(op.n)
        y = run_plan(P, x, rng=np.random.default_rng(seed + 10))
        assert rel(y, h2_matvec_ref(op, x)) <= 1e-13


@pytest.mark.parametrize("world", [1, 2, 4])
def test_level_skipping_chain(golden, world):
    """The level-skipping far-field chain (H2B_PLAN_SKIP_LEVELS): even-height
    clusters' x^ from the grandchildren through (F_g F_c)^T, every other
    level's y^ from the grandparent through E_c E_p -- the same product to
    rounding, with a chain of about half the links."""
    from oracle.flat_matvec import run_ranks
    from paper_1811_05731_b200.h2 import PLAN_SKIP_LEVELS, plan_view
    name, op, ex = golden
    plans = [plan_view(op, world_size=world, rank=r, plan_flags=PLAN_SKIP_LEVELS | PLAN_NO_STAGED) for r in range(world)]
    for i in (0, 3):
        y = run_ranks(plans, ex["X"][:, i]) if world > 1 else run_plan(plans[0], ex["X"][:, i])
        assert rel(y, ex["y_full"][:, i]) <= 1e-13, (name, world, i)
    if world == 1:
        check_plan_invariants(plans[0])
        base = plan_view(op, plan_flags=PLAN_NO_STAGED)
        assert plans[0]["stats"]["extra_bytes"] >= 0
        assert chain_length(plans[0]) <= chain_length(base)
        if chain_length(base) >= 8:   # deep enough for skipped links (config 1: 9 -> 7 items)
            assert chain_length(plans[0]) < chain_length(base), (chain_length(plans[0]), chain_length(base))


def chain_length(plan):
    """Longest dependency path (items) of a single-GPU plan."""
    T = len(plan["t_m"])
    depth = np.zeros(T, np.int64)
    for t in range(T):
        d = plan["deps"][plan["t_dep0"][t]:plan["t_dep0"][t + 1]]
        depth[t] = 1 + (depth[d].max() if d.size else 0)
    return int(depth.max())


@pytest.mark.parametrize("world", [1, 2, 4])
def test_gated_coupling_rows(golden, world):
    """H2B_PLAN_GATE: coupling rows fed only by upward coefficients lose their
    per-source dependencies and wait for the whole upward pass instead; the
    interpreter releases them exactly so (random dependency orders too)."""
    from oracle.flat_matvec import run_ranks
    from paper_1811_05731_b200.h2 import PLAN_GATE, plan_view
    name, op, ex = golden
    plans = [plan_view(op, world_size=world, rank=r, plan_flags=PLAN_GATE | PLAN_NO_STAGED) for r in range(world)]
    for i in (0, 2):
        y = run_ranks(plans, ex["X"][:, i]) if world > 1 else run_plan(plans[0], ex["X"][:, i])
        assert rel(y, ex["y_full"][:, i]) <= 1e-13, (name, world, i)
    if world == 1:
        p0 = plans[0]
        base = plan_view(op, plan_flags=0x200 | PLAN_NO_STAGED)   # no gate
        if len(op.coupling):
            assert p0["gated"].size > 0 and p0["ndeps"] < base["ndeps"] if "ndeps" in p0 else p0["gated"].size > 0
        assert np.all(p0["t_kind"][p0["gated"]] == 2)
        for g in p0["gated"]:
            assert p0["t_dep0"][g] == p0["t_dep0"][g + 1]
        rng = np.random.default_rng(5)
        for _ in range(2):
            coef = np.full((max(1, p0["coef_len"]), 1), np.nan)
            Y = np.full((op.n, 1), np.nan)
            from oracle.flat_matvec import run_phase
            run_phase(p0, ex["X"][:, 0], coef, Y, rng=rng)
            assert rel(Y[:, 0], ex["y_full"][:, 0]) <= 1e-13
