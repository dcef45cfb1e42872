"""Operator builder (the host-side producer of the matvec's input).

With the CPU restatement of the collocation entries the builder reproduces
the reference's H² operators bit for bit (tree, block lists, ranks, every
matrix); with the GPU collocation kernel the entries agree to rounding."""

import math

import numpy as np
import pytest

from conftest import load_golden, rel
from oracle.colloc_ref import CpuCollocation, panel_rows
from oracle.h2_matvec_ref import h2_matvec_ref
from paper_1811_05731_b200.assembly import geometry as G
from paper_1811_05731_b200.assembly.hbuild import CompressionConfig, assemble_h2


def _surface(ex):
    return G.make_surface(ex["boundary_coords"], ex["surface_triangles"],
                          psi=(ex["diag"] + 1.0) * 4.0 * math.pi)


def _cfg(ex):
    c = ex["config"]
    return CompressionConfig(leaf_size=int(c[0]), eta=float(c[1]), cheb_order=int(c[2]),
                             eps=float(c[3]), eps_rec=float(c[4]))


@pytest.mark.parametrize("name", ["sphere2_default", "sphere3_l32_eta2_o4", "torus_32_16_4_default"])
def test_builder_reproduces_reference_operator(name):
    ref, ex = load_golden(name)
    op, rep = assemble_h2(_surface(ex), _cfg(ex), evaluator=CpuCollocation, workers=2)
    assert np.array_equal(op.tree.perm, ref.tree.perm)
    assert [(a, b) for a, b, _ in op.coupling] == [(a, b) for a, b, _ in ref.coupling]
    assert [(a, b) for a, b, _ in op.near] == [(a, b) for a, b, _ in ref.near]
    for (_, _, m1), (_, _, m2) in zip(op.near, ref.near):
        assert np.array_equal(m1, m2)
    for (_, _, m1), (_, _, m2) in zip(op.coupling, ref.coupling):
        assert np.array_equal(m1, m2)
    assert op.storage_bytes() == ref.storage_bytes()
    assert np.array_equal(h2_matvec_ref(op, ex["X"][:, 0]), ex["y_full"][:, 0])


def test_icosphere_surface_is_reference_boundary():
    _, ex = load_golden("config1_sphere4")
    s = G.icosphere_surface(4)
    assert np.array_equal(s.coords, ex["boundary_coords"])
    assert np.array_equal(s.triangles, ex["surface_triangles"])
    assert np.abs(s.diag - ex["diag"]).max() < 1e-13   # dihedral vs tet solid angles


def test_solid_angles_cube():
    s = G.cube_surface(3)
    vals = np.unique(np.round(s.solid_angles / math.pi, 12))
    assert list(vals) == [0.5, 1.0, 2.0]


def test_row_sum_identity_small_cube():
    # closed-surface identity of the dense operator: M 1 = -1 (test_bem.py:96-102)
    s = G.cube_surface(3)
    ev = CpuCollocation(s, G.panel_table(s), G.incidence(s))
    n = s.n
    out = ev.rows(s.coords, np.zeros(n, np.int64), np.full(n, n, np.int32), np.arange(n),
                  np.arange(n) * n, np.arange(n), n * n)
    m = out.reshape(n, n)
    assert np.abs(m.sum(axis=1) + 1.0).max() < 1e-10


def test_generators_closed_and_sized():
    c = G.cube_surface(10)
    assert c.n == 6 * 100 + 2 and c.triangles.shape[0] == 2 * 6 * 100
    d = G.disk_surface(0.05)
    assert d.areas.min() > 0 and abs(d.areas.sum() - (2 * math.pi + 2 * math.pi * 0.05)) < 0.05
    assert np.all(d.solid_angles > 0) and np.all(d.solid_angles < 4 * math.pi)


@pytest.mark.gpu
def test_gpu_collocation_matches_cpu_restatement():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1811_05731_b200.assembly.hbuild import GpuCollocation
    s = G.disk_surface(0.05)
    pan, inc = G.panel_table(s), G.incidence(s)
    gpu = GpuCollocation(s, pan, inc)
    cpu = CpuCollocation(s, pan, inc)
    rng = np.random.default_rng(0)
    J = 300
    pts = np.concatenate([s.coords[rng.integers(0, s.n, J // 2)], rng.uniform(-1.2, 1.2, (J - J // 2, 3))])
    cnt = rng.integers(1, 80, J).astype(np.int32)
    cb = rng.integers(0, s.n - 80, J)
    dn = np.where(np.arange(J) < J // 2, rng.integers(0, s.n, J), -1)
    off = np.concatenate([[0], np.cumsum(cnt)[:-1]])
    colidx = rng.permutation(s.n)
    a = gpu.rows(pts, cb, cnt, dn, off, colidx, int(cnt.sum()))
    b = cpu.rows(pts, cb, cnt, dn, off, colidx, int(cnt.sum()))
    assert np.abs(a - b).max() <= 1e-13 * np.abs(b).max()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["sphere3_l32_eta2_o4", "config1_sphere4"])
def test_gpu_built_operator_matches_reference(name):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ref, ex = load_golden(name)
    op, rep = assemble_h2(_surface(ex), _cfg(ex), workers=4)
    assert np.array_equal(op.tree.perm, ref.tree.perm)
    assert [(a, b) for a, b, _ in op.near] == [(a, b) for a, b, _ in ref.near]
    assert max(np.abs(m1 - m2).max() for (_, _, m1), (_, _, m2) in zip(op.near, ref.near)) < 1e-14
    # entries differ from the reference only by rounding: same accuracy
    for i in range(3):
        assert rel(h2_matvec_ref(op, ex["X"][:, i]), ex["y_full"][:, i]) <= 1e-9


@pytest.mark.parametrize("name", ["sphere3_l32_eta2_o4", "torus_32_16_4_default"])
def test_batched_hca_backend_same_operator_to_compression_accuracy(name):
    """backend="gpu" (batched HCA, Gram-based bases; run here on torch's CPU
    device) builds the same operator as the reference up to rounding at the
    truncation thresholds: same blocks, products within the compression
    accuracy of each other and of the dense operator."""
    ref, ex = load_golden(name)
    op, rep = assemble_h2(_surface(ex), _cfg(ex), evaluator=CpuCollocation, workers=2, backend="gpu",
                          device="cpu")
    assert [(a, b) for a, b, _ in op.coupling] == [(a, b) for a, b, _ in ref.coupling]
    assert [(a, b) for a, b, _ in op.near] == [(a, b) for a, b, _ in ref.near]
    assert abs(op.storage_bytes() - ref.storage_bytes()) <= 0.02 * ref.storage_bytes()
    for i in range(3):
        y = h2_matvec_ref(op, ex["X"][:, i])
        assert rel(y, ex["y_full"][:, i]) <= 1e-4
        assert rel(y, ex["y_dense"][:, i]) <= 2.0 * rel(ex["y_full"][:, i], ex["y_dense"][:, i]) + 1e-5


@pytest.mark.gpu
def test_batched_hca_on_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ref, ex = load_golden("config1_sphere4")
    op, rep = assemble_h2(_surface(ex), _cfg(ex), workers=4, backend="gpu")
    assert [(a, b) for a, b, _ in op.coupling] == [(a, b) for a, b, _ in ref.coupling]
    for i in range(3):
        y = h2_matvec_ref(op, ex["X"][:, i])
        assert rel(y, ex["y_full"][:, i]) <= 1e-4
        assert rel(y, ex["y_dense"][:, i]) <= 2.0 * rel(ex["y_full"][:, i], ex["y_dense"][:, i]) + 1e-5
