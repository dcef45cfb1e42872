"""Staged product (H2B_PLAN_STAGED): upward sweep over the
bottom subtrees, one dataflow launch (near field, coupling rows, the chain of
the clusters above the subtrees), downward sweep with the finals.  The numpy
interpreter executes every launch the way its kernel does -- a sweep's waves
against a snapshot of the workspace, so an item reading what another item of
its wave writes would be caught -- and must reproduce the reference."""

import dataclasses

import numpy as np
import pytest

from conftest import load_golden, rel
from oracle.flat_matvec import check_plan_invariants, launches, run_plan, run_ranks
from oracle.h2_matvec_ref import h2_matvec_ref
from paper_1811_05731_b200.h2 import (PLAN_NEAR_SPLIT, PLAN_NO_SKIP, PLAN_SKIP_LEVELS, PLAN_STAGED,
                                      PLAN_SWEEP_NODES, plan_view)
from synth import random_h2


@pytest.mark.parametrize("nodes", [0, 1, 2, 3, 8])
def test_staged_plan_matches_reference(golden, nodes):
    name, op, ex = golden
    P = plan_view(op, plan_flags=PLAN_STAGED | PLAN_SWEEP_NODES(nodes))
    check_plan_invariants(P)
    modes = [ph["mode"] for ph in launches(P)]
    assert modes.count(0) == 1 and modes[-1] == 1          # ... dataflow ... down sweep (the finals)
    if len(op.coupling):
        assert modes == [1, 0, 1]
    assert P["stats"]["stream_bytes"] == int(ex["storage_bytes"])
    for i in (0, 2):
        assert rel(run_plan(P, ex["X"][:, i]), ex["y_full"][:, i]) <= 1e-13, (name, nodes, i)
    y = run_plan(P, ex["X"][:, 1], rng=np.random.default_rng(nodes))
    assert rel(y, ex["y_full"][:, 1]) <= 1e-13, (name, nodes)


def test_staged_sweeps_hold_the_subtrees_and_the_rest_has_no_finals(golden):
    name, op, ex = golden
    P = plan_view(op, plan_flags=PLAN_STAGED | PLAN_SWEEP_NODES(2) | PLAN_NO_SKIP)
    up, flow, down = launches(P) if len(op.coupling) else (None, launches(P)[0], launches(P)[-1])
    nleaves = sum(1 for c in op.tree.clusters if c.is_leaf)
    assert int((down["t_kind"] == 4).sum()) == nleaves and not (flow["t_kind"] == 4).any()
    if up is not None:
        assert np.all(up["t_kind"] <= 1) and len(up["deps"]) == 0
        # every leaf's forward transform is in the upward sweep
        assert not (flow["t_kind"] == 0).any()
    # a unit's waves are contiguous and tile the launch
    for sw in (s for s in (up, down) if s is not None):
        assert sw["wave0"][0] == 0 and np.all(np.diff(sw["wave0"]) > 0)
        assert np.all(np.diff(sw["unit0"]) > 0)


def test_staged_ablations(golden):
    name, op, ex = golden
    x = ex["X"][:, 0]
    for abl, key in ((dataclasses.replace(op, coupling=[]), "y_near"),
                     (dataclasses.replace(op, near=[]), "y_far")):
        y = run_plan(plan_view(abl, plan_flags=PLAN_STAGED | PLAN_SWEEP_NODES(2)), x)
        assert rel(y, ex[key][:, 0]) <= 1e-13, (name, key)


@pytest.mark.parametrize("skip", [PLAN_SKIP_LEVELS, PLAN_NO_SKIP])
def test_staged_with_level_skipping_above_the_subtrees(golden, skip):
    name, op, ex = golden
    P = plan_view(op, plan_flags=PLAN_STAGED | PLAN_SWEEP_NODES(1) | skip)
    check_plan_invariants(P)
    if skip == PLAN_NO_SKIP:
        assert P["stats"]["extra_bytes"] == 0
    for seed in range(2):
        y = run_plan(P, ex["X"][:, 3], rng=np.random.default_rng(seed))
        assert rel(y, ex["y_full"][:, 3]) <= 1e-13, (name, skip)


@pytest.mark.parametrize("seed", range(4))
def test_staged_random_structures(seed):
    op = random_h2(seed)
    x = np.random.default_rng(seed).standard_normal((op.n, 2))
    for flags in (PLAN_STAGED, PLAN_STAGED | PLAN_SWEEP_NODES(1), PLAN_STAGED | PLAN_SWEEP_NODES(2) | PLAN_SKIP_LEVELS):
        P = plan_view(op, plan_flags=flags, task_bytes=700)
        check_plan_invariants(P)
        Y = run_plan(P, x, rng=np.random.default_rng(seed + 1))
        for i in range(2):
            assert rel(Y[:, i], h2_matvec_ref(op, x[:, i])) <= 1e-13, (seed, flags)


def test_staged_split_product(golden):
    """The split multi-RHS product planned beside a staged plan keeps every
    far-field item in its dataflow launch (sweeps of 8/16 right-hand sides
    measured slower): the near field alone, then the rest."""
    name, op, ex = golden
    P = plan_view(op, plan_flags=PLAN_STAGED | PLAN_SWEEP_NODES(2) | PLAN_NEAR_SPLIT)
    sp = launches(P, split=True)
    assert [ph["mode"] for ph in sp] == [2, 0]
    assert np.all(sp[0]["t_kind"] == 3) and int((sp[1]["t_kind"] == 4).sum()) > 0
    Y = run_plan(P, ex["X"][:, :4], split=True)
    for i in range(4):
        assert rel(Y[:, i], ex["y_full"][:, i]) <= 1e-13, (name, i)


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_staged_rank_plans(golden, world):
    """Ranks own whole bottom subtrees: sweep, dataflow (the owned upper
    clusters and the phase-0 near field), exchange, dataflow, sweep."""
    name, op, ex = golden
    plans = [plan_view(op, world_size=world, rank=r, plan_flags=PLAN_STAGED | PLAN_SWEEP_NODES(2))
             for r in range(world)]
    lohi = plans[0]["rank_lo_hi"]
    assert lohi[0, 0] == 0 and lohi[-1, 1] == op.n and np.all(lohi[1:, 0] == lohi[:-1, 1])
    for i in (0, 4):
        assert rel(run_ranks(plans, ex["X"][:, i]), ex["y_full"][:, i]) <= 1e-13, (name, world, i)
    for p in plans:
        assert p["stats"]["pool_bytes"] == p["stats"]["local_bytes"]


@pytest.mark.parametrize("seed", range(3))
def test_staged_rank_plans_random_structures(seed):
    op = random_h2(seed)
    x = np.random.default_rng(seed).standard_normal(op.n)
    ref = h2_matvec_ref(op, x)
    for world in (2, 5):
        plans = [plan_view(op, world_size=world, rank=r, plan_flags=PLAN_STAGED) for r in range(world)]
        assert rel(run_ranks(plans, x), ref) <= 1e-13


def test_staged_units_are_contiguous_ranges(golden):
    """Resident sweeps: a unit's matrices, coefficient slots, near-field
    partial slots and x range are contiguous, cover exactly what its items
    touch inside the subtree, and units do not overlap."""
    name, op, ex = golden
    P = plan_view(op, plan_flags=PLAN_STAGED | PLAN_SWEEP_NODES(2))
    for ph in launches(P):
        if ph["mode"] != 1:
            continue
        assert ph["resident"], name
        R = ph["u_range"]
        up = ph["t_kind"][0] <= 1
        assert np.all(R[:, 1::2] >= 0)
        for col in (0, 2, 4):           # pool, coefficient and partial ranges of different units are disjoint
            o = np.argsort(R[:, col], kind="stable")
            lo, ln = R[o, col], R[o, col + 1]
            assert np.all(lo[1:] >= (lo + ln)[:-1]), (name, col)
        for u in range(len(R)):
            k0, k1 = ph["wave0"][ph["unit0"][u]], ph["wave0"][ph["unit0"][u + 1]]
            for t in range(k0, k1):
                d0 = ph["t_data"][t]
                last = d0 + (ph["t_ncols"][t] - 1) * ph["t_ld"][t] + ph["t_m"][t]
                assert R[u, 0] <= d0 and last <= R[u, 0] + R[u, 1], (name, u, t)
                if ph["t_kind"][t] != 4:   # outputs stay inside the unit's main coefficient range
                    assert R[u, 2] <= ph["t_out"][t] and ph["t_out"][t] + ph["t_m"][t] <= R[u, 2] + R[u, 3]
                else:
                    assert R[u, 6] <= ph["t_out"][t] and ph["t_out"][t] + ph["t_m"][t] <= R[u, 6] + R[u, 7]
                    if ph["t_bias"][t] >= 0:
                        assert R[u, 4] <= ph["t_bias"][t] < R[u, 4] + R[u, 5]
            if up:
                assert R[u, 5] == 0
