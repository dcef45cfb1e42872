"""The solve either side of the boundary operator: the
GPU Jacobi-PCG (csrc/cg.cu, ``paper_1811_05731_b200.fem.cg_solve``, the
drop-in for solver.py:44-98) against the oracle's CG on the same systems,
and the reference's own pipeline (``strayfield.pipeline.compute_demag``,
pipeline.py:46-63, from baseline/_ref) run with BOTH GPU drop-ins installed
into the reference modules.

CG tolerance: the GPU sums the dot products in a different order than
numpy, so iterates agree to the solve tolerance (tol = 1e-10 relative
residual), not bit for bit; the energy of the uniformly magnetized sphere
is compared at 1e-9 relative, the iteration counts to within 2.
"""

import numpy as np
import pytest

from conftest import ROOT, load_golden, rel

gpu = pytest.mark.gpu


def _mesh():
    from oracle.mesh_ref import generate_sphere_mesh
    return generate_sphere_mesh(1.0, 4)


def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()


def test_precond_contract_cpu():
    """Only the Jacobi preconditioner runs on the GPU (no CPU fallback);
    the check itself needs no GPU."""
    from scipy.sparse import diags
    from paper_1811_05731_b200 import fem
    a = diags([2.0, 3.0, 4.0]).tocsr()
    inv = 1.0 / a.diagonal()
    assert fem._is_jacobi(a, lambda r: inv * r)
    from oracle.reference import available, strayfield
    if available():   # the reference's own preconditioner object
        strayfield()
        from strayfield.solver import jacobi_preconditioner
        assert fem._is_jacobi(a, jacobi_preconditioner(a))
    assert not fem._is_jacobi(a, lambda r: r)
    with pytest.raises(NotImplementedError):
        fem.cg_solve(a, np.ones(3), precond=lambda r: r)


@gpu
@pytest.mark.parametrize("deflate", [True, False])
def test_gpu_cg_matches_oracle_cg(deflate):
    _cuda()
    from oracle.fem_ref import _pcg, rhs_u1, stiffness
    from paper_1811_05731_b200 import fem
    mesh = _mesh()
    a = stiffness(mesh)
    rng = np.random.default_rng(5)
    if deflate:
        b = rhs_u1(mesh, rng.standard_normal((mesh.n_nodes, 3)))
        mat = a
    else:
        interior = np.setdiff1d(np.arange(mesh.n_nodes), mesh.boundary_nodes)
        mat = a[interior][:, interior].tocsr()
        b = rng.standard_normal(interior.size)
    x, rep = fem.cg_solve(mat, b, tol=1e-10, deflate_constants=deflate)
    xo, ito = _pcg(mat, b, 1e-10, deflate)
    assert rep.converged and rep.residual <= 1e-10
    assert abs(rep.iterations - ito) <= 2
    assert rel(x, xo) <= 1e-8
    bb = b - b.mean() if deflate else b
    assert np.linalg.norm(bb - mat @ x) <= 1.5e-10 * np.linalg.norm(b)
    if deflate:
        assert abs(x.mean()) <= 1e-14 * np.abs(x).max()


@gpu
def test_gpu_cg_contract():
    _cuda()
    from scipy.sparse import csr_matrix, diags
    from paper_1811_05731_b200 import fem
    a = diags([2.0, 3.0, 4.0]).tocsr()
    x, rep = fem.cg_solve(a, np.zeros(3))
    assert rep.iterations == 0 and np.array_equal(x, np.zeros(3))
    x, rep = fem.cg_solve(a, np.array([2.0, 3.0, 4.0]))
    assert np.allclose(x, 1.0) and rep.converged
    # max_iter <= 0: the reference's loop never runs (solver.py:80-90)
    x, rep = fem.cg_solve(a, np.array([2.0, 3.0, 4.0]), max_iter=0)
    assert np.array_equal(x, np.zeros(3)) and rep.iterations == 0 and rep.residual == 1.0 and not rep.converged
    with pytest.raises(ValueError, match="zero-free diagonal"):
        fem.GpuCG(csr_matrix(np.array([[0.0, 1.0], [1.0, 2.0]])))
    with pytest.raises(ValueError, match="incompatible rhs"):
        fem.cg_solve(a, np.array([1.0, 1.0, 1.0]), deflate_constants=True)
    with pytest.raises(fem.ConvergenceError, match="negative curvature"):
        fem.cg_solve(diags([-1.0, -2.0]).tocsr(), np.array([1.0, 1.0]))


@gpu
@pytest.mark.skipif(not (ROOT / "baseline" / "_ref" / "strayfield").exists(),
                    reason="baseline/_ref not vendored (tools/vendor_reference.sh)")
def test_reference_pipeline_with_gpu_solves_and_product():
    """The reference's compute_demag (pipeline.py:46-63) on its own sphere
    mesh, with ``solver.cg_solve`` and ``h2_matvec`` both routed to the GPU,
    matches the reference energy e_d/K_d = 0.3329597004200991 (config 1)."""
    _cuda()
    import sys
    from oracle.reference import strayfield
    strayfield()
    from strayfield import fem as rfem, mesh as rmesh, pipeline as rpipe, solver as rsolver
    import strayfield.hmatrix as rhm
    import strayfield.hmatrix.h2 as rh2
    from oracle.reference import to_reference
    from paper_1811_05731_b200 import fem, h2
    saved = (rsolver.cg_solve, rfem.cg_solve, rh2.h2_matvec, rhm.h2_matvec)
    calls = {"cg": 0, "h2": 0}
    try:
        fem.install_into_reference(rsolver, rfem)
        h2.install_into_reference(rh2, rhm)
        gpu_cg, gpu_h2 = rfem.cg_solve, rh2.h2_matvec

        def cg_counted(*a, **k):
            calls["cg"] += 1
            return gpu_cg(*a, **k)

        def h2_counted(op, x):
            calls["h2"] += 1
            return gpu_h2(op, x)

        rfem.cg_solve, rh2.h2_matvec = cg_counted, h2_counted
        op, ex = load_golden("config1_sphere4")
        mesh = rmesh.generate_sphere_mesh(1.0, 4)
        from strayfield.bem import BoundaryOperator
        bop = BoundaryOperator(backend="h2", n=op.n, diag=np.zeros(op.n), payload=to_reference(op))
        m = rpipe.magnetization_preset(mesh, "uniform-z")
        res = rpipe.compute_demag(mesh, m, bop)
    finally:
        rsolver.cg_solve, rfem.cg_solve, rh2.h2_matvec, rhm.h2_matvec = saved
    assert calls == {"cg": 2, "h2": 1}
    ref = float(ex["energy_e_d_over_kd"])
    assert abs(res.e_d_over_kd - ref) <= 1e-9 * abs(ref)
    assert abs(res.u1_iterations - 248) <= 2 and abs(res.u2_iterations - 217) <= 2
    assert rel(res.u2[mesh.boundary_nodes], ex["energy_u2_boundary"]) <= 1e-8


@gpu
@pytest.mark.skipif(not (ROOT / "baseline" / "_ref" / "strayfield").exists(),
                    reason="baseline/_ref not vendored (tools/vendor_reference.sh)")
def test_device_pipeline_matches_reference_pipeline():
    """``paper_1811_05731_b200.pipeline.compute_demag`` -- both solves and
    the H² product chained in device memory -- against the unmodified
    reference's compute_demag (pipeline.py:46-63) on the config-1 sphere:
    the energy to 1e-9, the potentials to the solve tolerance."""
    _cuda()
    from oracle.reference import strayfield, to_reference
    strayfield()
    from strayfield import fem as rfem, mesh as rmesh, pipeline as rpipe
    from strayfield.bem import BoundaryOperator
    from paper_1811_05731_b200 import pipeline
    op, ex = load_golden("config1_sphere4")
    mesh = rmesh.generate_sphere_mesh(1.0, 4)
    bop = BoundaryOperator(backend="h2", n=op.n, diag=np.zeros(op.n), payload=to_reference(op))
    m = rpipe.magnetization_preset(mesh, "uniform-z")
    want = rpipe.compute_demag(mesh, m, bop)          # the reference, on the CPU
    got = pipeline.compute_demag(mesh, m, bop, fem=rfem)
    assert isinstance(got, rpipe.PipelineResult)
    ref = float(ex["energy_e_d_over_kd"])
    assert abs(got.e_d_over_kd - ref) <= 1e-9 * abs(ref)
    assert abs(got.e_d_over_kd - want.e_d_over_kd) <= 1e-9 * abs(ref)
    assert abs(got.u1_iterations - want.u1_iterations) <= 2 and abs(got.u2_iterations - want.u2_iterations) <= 2
    assert rel(got.u1, want.u1) <= 1e-8 and rel(got.u2, want.u2) <= 1e-8 and rel(got.u, want.u) <= 1e-8
    assert got.h_field.shape == want.h_field.shape and rel(got.h_field, want.h_field) <= 1e-7
    # contract: only the H² backend runs on the device
    dense = BoundaryOperator(backend="dense", n=op.n, diag=np.zeros(op.n), payload=np.eye(op.n))
    with pytest.raises(NotImplementedError):
        pipeline.compute_demag(mesh, m, dense, fem=rfem)


@gpu
def test_gpu_cg_kernel_variants(monkeypatch):
    """Every kernel variant of csrc/cg.cu (H2B_CG_VARIANT, read when the
    solver is created) solves the same system to the oracle's solution.
    Variants with the same grid sum in the same order: <2,4,256> and
    <1,4,256> (592 CTAs), and <2,2,512> with and without the L2 prefetch,
    give bit-identical iterates."""
    _cuda()
    from oracle.fem_ref import _pcg, rhs_u1, stiffness
    from paper_1811_05731_b200 import fem
    mesh = _mesh()
    a = stiffness(mesh)
    b = rhs_u1(mesh, np.random.default_rng(9).standard_normal((mesh.n_nodes, 3)))
    xo, ito = _pcg(a, b, 1e-10, True)
    out = {}
    for v in range(7):
        for rp_smem in ("1", "0"):
            monkeypatch.setenv("H2B_CG_VARIANT", str(v))
            monkeypatch.setenv("H2B_CG_RP_SMEM", rp_smem)
            solver = fem.GpuCG(a)
            x, rep = solver.solve(b, deflate_constants=True)
            assert rep.converged and abs(rep.iterations - ito) <= 2, (v, rp_smem)
            assert rel(x, xo) <= 1e-8, (v, rp_smem)
            out[v, rp_smem] = x
    for v in range(7):
        # the row pointers' location changes no arithmetic (L2 prefetch off without them)
        assert np.array_equal(out[v, "1"], out[v, "0"]), v
    assert np.array_equal(out[0, "1"], out[3, "1"])
    assert np.array_equal(out[4, "1"], out[6, "1"])
