"""``compute_demag`` with the whole potential split on the device
(SURVEY §8f row 3's end state; pipeline.py:46-63, fem.py:79-121).

The reference runs  u1 = solve_u1(...)  ->  u2|boundary = M u1|boundary  ->
u2 = solve_u2(...)  ->  u = u1 + u2  with numpy arrays between the steps.
With the drop-ins installed one at a time (``fem.install_into_reference``,
``h2.install_into_reference``) each step round-trips its vectors through host
memory.  Here the three steps are chained on the GPU: the right-hand side of
u1 goes up once, the Jacobi-PCG (``h2b_cg_solve_dev``) leaves u1 in HBM, the
boundary values are gathered there, the H² product (``h2b_matvec_dev``) and
the second solve read and write device memory, and u1, u2, u come down once.

The FEM assembly, the field and the energy are the reference's own functions
(out of scope): pass the reference's ``fem`` module (default:
``strayfield.fem`` if importable).  The result type is the reference's
``PipelineResult`` when its ``pipeline`` module is given or importable.
There is no CPU fallback: a non-"h2" operator raises.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .fem import GpuCG
from .h2 import device_operator

__all__ = ["compute_demag", "PipelineResult"]


@dataclass(frozen=True)
class PipelineResult:  # pipeline.py:34-43
    u1: np.ndarray
    u2: np.ndarray
    u: np.ndarray
    h_field: np.ndarray
    e_d: float
    e_d_over_kd: float
    u1_iterations: int
    u2_iterations: int


def compute_demag(mesh, m_nodal, operator, tol: float = 1e-10, *, fem=None, result_type=None):
    """pipeline.py:46-63 with solve_u1, the boundary operator and solve_u2 on
    the device.  ``mesh``/``m_nodal``/``operator`` as the reference takes
    them (a ``BoundaryOperator`` whose backend is "h2")."""
    import torch
    if fem is None:
        from strayfield import fem  # the reference's assembly, field and energy
    if getattr(operator, "backend", None) != "h2":
        raise NotImplementedError("the device pipeline applies the H² boundary operator (backend 'h2')")
    if result_type is None:
        try:
            from strayfield.pipeline import PipelineResult as result_type
        except ImportError:
            result_type = PipelineResult
    dev = torch.device("cuda")
    n = int(mesh.n_nodes)
    bnodes = np.asarray(mesh.boundary_nodes, np.int64)
    if operator.n != bnodes.size:
        raise ValueError(f"operator has {operator.n} boundary nodes, the mesh {bnodes.size}")
    stiffness = fem.assemble_stiffness(mesh)
    # --- u1: singular Neumann problem, constant mode deflated (fem.py:79-95)
    b = np.ascontiguousarray(fem.assemble_u1_rhs(mesh, m_nodal), np.float64)
    if np.linalg.norm(b) == 0.0:
        u1_d, it1 = torch.zeros(n, dtype=torch.float64, device=dev), 0
    else:
        if abs(b.sum()) > 1e-10 * np.abs(b).sum():  # solver.py:68-70
            raise ValueError("incompatible rhs: not orthogonal to the constant kernel")
        cg1 = GpuCG(stiffness)
        try:
            u1_d, rep1 = cg1.solve_dev(torch.from_numpy(b).to(dev), tol=tol, deflate_constants=True)
        finally:
            cg1.close()
        it1 = rep1.iterations
    # --- boundary operator: u2|boundary = M u1|boundary (pipeline.py:54, bem.py:272-284)
    bn_d = torch.from_numpy(bnodes).to(dev)
    xb = u1_d.index_select(0, bn_d).contiguous()
    yb = torch.empty_like(xb)
    dop = device_operator(operator.payload)
    dop.matvec_dev(xb.data_ptr(), yb.data_ptr(), 1, torch.cuda.current_stream().cuda_stream)
    # --- u2: Laplace problem with Dirichlet data (fem.py:98-121)
    u2_d = torch.zeros(n, dtype=torch.float64, device=dev)
    u2_d[bn_d] = yb
    interior = np.setdiff1d(np.arange(n), bnodes)
    it2 = 0
    if interior.size:
        a_int = stiffness[interior]
        a_ii = a_int[:, interior].tocsr()
        a_ib = a_int[:, bnodes].tocsr()      # u is zero off the boundary: rhs = -(a[interior] @ u) = -a_ib yb
        a_ib_d = torch.sparse_csr_tensor(torch.from_numpy(a_ib.indptr.astype(np.int64)),
                                         torch.from_numpy(a_ib.indices.astype(np.int64)),
                                         torch.from_numpy(np.ascontiguousarray(a_ib.data, np.float64)),
                                         size=a_ib.shape).to(dev)
        rhs = -(a_ib_d @ yb)
        cg2 = GpuCG(a_ii)
        try:
            x_d, rep2 = cg2.solve_dev(rhs, tol=tol)
        finally:
            cg2.close()
        it2 = rep2.iterations
        u2_d[torch.from_numpy(interior).to(dev)] = x_d
    u_d = u1_d + u2_d
    u1, u2, u = (t.cpu().numpy() for t in (u1_d, u2_d, u_d))
    h = fem.compute_field(mesh, u)
    e_d, e_ratio = fem.magnetostatic_energy(mesh, m_nodal, h)
    return result_type(u1=u1, u2=u2, u=u, h_field=h, e_d=e_d, e_d_over_kd=e_ratio,
                       u1_iterations=it1, u2_iterations=it2)
