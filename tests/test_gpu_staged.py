"""GPU parity of the staged product: sweep kernels over the
bottom subtrees around one dataflow launch, through the C ABI, against the
reference's outputs and the oracle (relative l2 <= 1e-12, fp64)."""

import dataclasses

import numpy as np
import pytest

from conftest import load_golden, rel
from oracle.h2_matvec_ref import h2_matvec_ref
from synth import random_h2

pytestmark = pytest.mark.gpu
TOL = 1e-12


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()


def _h2():
    from paper_1811_05731_b200 import h2
    return h2


STREAMING = dict(sched_flags=8 | (8 << 4) | (2 << 18) | (6 << 26) | (4 << 20) | (1 << 25), task_bytes=262144)


@pytest.mark.parametrize("nodes", [0, 1, 2, 4])
@pytest.mark.parametrize("opts", [{}, STREAMING, dict(task_bytes=700, far_task_bytes=512)])
def test_staged_full_product(golden, nodes, opts):
    name, op, ex = golden
    h2 = _h2()
    dev = h2.DeviceOperator(op, plan_flags=h2.PLAN_STAGED | h2.PLAN_SWEEP_NODES(nodes), **opts)
    try:
        for _ in range(2):   # twice: nothing may be left over from the first product
            for i in range(ex["X"].shape[1]):
                assert rel(dev.matvec(ex["X"][:, i]), ex["y_full"][:, i]) <= TOL, (name, nodes, i)
    finally:
        dev.close()


def test_staged_far_and_near_fields_separately(golden):
    name, op, ex = golden
    h2 = _h2()
    x = ex["X"][:, 0]
    for abl, key in ((dataclasses.replace(op, near=[]), "y_far"), (dataclasses.replace(op, coupling=[]), "y_near")):
        if key == "y_far" and not op.coupling:
            continue
        dev = h2.DeviceOperator(abl, plan_flags=h2.PLAN_STAGED | h2.PLAN_SWEEP_NODES(2))
        try:
            assert rel(dev.matvec(x), ex[key][:, 0]) <= TOL, (name, key)
        finally:
            dev.close()


@pytest.mark.parametrize("nrhs", [2, 4, 8, 16])
@pytest.mark.parametrize("name", ["config1_sphere4", "prism_20_40_2_default"])
def test_staged_multi_rhs(name, nrhs):
    op, ex = load_golden(name)
    h2 = _h2()
    X = np.random.default_rng(nrhs).standard_normal((op.n, nrhs))
    dev = h2.DeviceOperator(op, plan_flags=h2.PLAN_STAGED | h2.PLAN_SWEEP_NODES(2))
    try:
        Y = dev.matvec(X)
    finally:
        dev.close()
    for i in range(nrhs):
        assert rel(Y[:, i], h2_matvec_ref(op, X[:, i])) <= TOL, (name, nrhs, i)


@pytest.mark.parametrize("seed", range(4))
def test_staged_random_structures(seed):
    """Adversarial structures: ranks and leaves above 64 (row tiles), rank-0
    clusters, non-leaf near blocks, heavy rows."""
    op = random_h2(seed)
    h2 = _h2()
    X = np.random.default_rng(seed).standard_normal((op.n, 4))
    for flags in (h2.PLAN_STAGED, h2.PLAN_STAGED | h2.PLAN_SWEEP_NODES(1) | h2.PLAN_SKIP_LEVELS):
        dev = h2.DeviceOperator(op, plan_flags=flags, task_bytes=700)
        try:
            y = dev.matvec(X[:, 0])
            Y = dev.matvec(X)
        finally:
            dev.close()
        assert rel(y, h2_matvec_ref(op, X[:, 0])) <= TOL, (seed, flags)
        for i in range(4):
            assert rel(Y[:, i], h2_matvec_ref(op, X[:, i])) <= TOL, (seed, flags, i)


def test_staged_is_deterministic_and_linear():
    op, ex = load_golden("torus_32_16_4_default")
    h2 = _h2()
    dev = h2.DeviceOperator(op, plan_flags=h2.PLAN_STAGED | h2.PLAN_SWEEP_NODES(2))
    try:
        x, z = ex["X"][:, 0], ex["X"][:, 1]
        y1, y2 = dev.matvec(x), dev.matvec(x)
        assert np.array_equal(y1, y2)
        assert np.array_equal(dev.matvec(np.zeros(op.n)), np.zeros(op.n))
        lin = dev.matvec(2.0 * x - 0.5 * z)
        assert rel(lin, 2.0 * y1 - 0.5 * dev.matvec(z)) <= 1e-13
    finally:
        dev.close()


@pytest.mark.parametrize("world", [2, 4])
def test_staged_virtual_ranks_on_one_gpu(world):
    """The ranks of a staged multi-GPU product one after another on one
    device: group 0 of every rank (upward sweep of its subtrees, then the
    owned upper clusters and its phase-0 near field), the region copies,
    group 1 (dataflow launch, downward sweep)."""
    import torch
    h2 = _h2()
    for name in ("config1_sphere4", "prism_20_40_2_default"):
        op, ex = load_golden(name)
        opts = dict(plan_flags=h2.PLAN_STAGED | h2.PLAN_SWEEP_NODES(1))
        devs = [h2.DeviceOperator(op, world_size=world, rank=r, **opts) for r in range(world)]
        x = torch.from_numpy(ex["X"][:, 0]).cuda()
        ys = [torch.zeros_like(x) for _ in range(world)]
        s = torch.cuda.current_stream().cuda_stream
        for _ in range(2):
            for r, d in enumerate(devs):
                d.matvec_phase(0, x.data_ptr(), ys[r].data_ptr(), 1, s)
            for r, d in enumerate(devs):
                for q, o in enumerate(devs):
                    if q != r:
                        d.exchange_copy_from(o, 1, s)
            for r, d in enumerate(devs):
                d.matvec_phase(1, x.data_ptr(), ys[r].data_ptr(), 1, s)
            torch.cuda.synchronize()
            plans = [h2.plan_view(op, world_size=world, rank=r, **opts) for r in range(world)]
            y = np.zeros(op.n)
            for r in range(world):
                lo, hi = plans[r]["rank_lo_hi"][r]
                rows = plans[r]["perm"][lo:hi]
                y[rows] = ys[r].cpu().numpy()[rows]
            assert rel(y, ex["y_full"][:, 0]) <= TOL, (name, world)
        for d in devs:
            d.close()


def test_resident_and_generic_sweeps_agree(monkeypatch):
    """The resident sweep kernel (units run from shared memory) and the
    generic one compute the same items; both match the reference, and the
    small golden operators fit shared memory for 1-4 right-hand sides."""
    h2 = _h2()
    for name in ("config1_sphere4", "torus_32_16_4_default"):
        op, ex = load_golden(name)
        ys = []
        for res in ("1", "0"):
            monkeypatch.setenv("H2B_SWEEP_RESIDENT", res)
            dev = h2.DeviceOperator(op, plan_flags=h2.PLAN_STAGED | h2.PLAN_SWEEP_NODES(2))
            try:
                mask = dev.stats()["resident_mask"]
                assert (mask & 1) == (1 if res == "1" else 0), (name, res, mask)
                ys.append(dev.matvec(ex["X"][:, 0]))
                Y = dev.matvec(ex["X"][:, :4])
                for i in range(4):
                    assert rel(Y[:, i], ex["y_full"][:, i]) <= TOL, (name, res, i)
            finally:
                dev.close()
        assert rel(ys[0], ex["y_full"][:, 0]) <= TOL and rel(ys[1], ex["y_full"][:, 0]) <= TOL
        assert rel(ys[0], ys[1]) <= 1e-14
