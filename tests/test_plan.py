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
from paper_1811_05731_b200.h2 import plan_view
from synth import random_h2


def test_abi_exports_every_declared_symbol():
    header = (ROOT / "include" / "h2b.h").read_text()
    names = re.findall(r"^\s*(?:int|void|int64_t|const char\*)\s+\**(h2b_\w+)\s*\(", header, re.M)
    assert len(names) >= 12
    lib = ctypes.CDLL(str(nat.LIB_PATH))
    for nm in names:
        assert hasattr(lib, nm), nm
    assert nat.lib().h2b_abi_version() == 1


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
    assert sum(st["bytes_by_kind"].values()) == st["stream_bytes"] == op.storage_bytes()
    assert st["tasks_by_kind"]["final"] == sum(1 for c in op.tree.clusters if c.is_leaf)
