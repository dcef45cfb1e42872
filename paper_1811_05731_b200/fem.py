"""The FEM steps either side of the boundary operator, with the solves on the
GPU.

Assembly stays on the host in numpy, as in the reference (fem.py:32-76,
124-146: tet gradients, P1 stiffness, the Neumann right-hand side, field and
energy).  The two solves -- the singular Neumann problem for u1 with the
constant mode deflated (fem.py:79-95) and the Dirichlet problem for u2 on
the interior block (fem.py:98-121) -- run the reference's
Jacobi-preconditioned CG (solver.py:44-98) as one cooperative CUDA kernel
(`csrc/cg.cu`, `h2b_cg_*` in include/h2b.h).  There is no CPU fallback: the
solves fail loudly without the library.

The mesh is duck-typed like the reference's ``TetMesh`` (``nodes``,
``tets``, ``boundary_nodes``, ``n_nodes``, ``n_boundary``).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
from scipy.sparse import coo_matrix, csr_matrix

from . import _native as nat

__all__ = ["SolveReport", "ConvergenceError", "GpuCG", "cg_solve", "tet_gradients", "assemble_stiffness",
           "assemble_u1_rhs", "solve_u1", "solve_u2", "compute_field", "magnetostatic_energy",
           "STRAY_FIELD_CONSTANT"]

STRAY_FIELD_CONSTANT = 0.5  # K_d = mu0 Ms^2 / 2 (fem.py:29)


class ConvergenceError(RuntimeError):
    """Iterative solver failed (errors.py ConvergenceError)."""


@dataclass(frozen=True)
class SolveReport:  # solver.py:20-24
    iterations: int
    residual: float
    converged: bool


class GpuCG:
    """A sparse symmetric matrix resident on the GPU with its Jacobi
    preconditioner (``h2b_cg``); ``solve`` runs cg_solve (solver.py:44-98)."""

    def __init__(self, a):
        a = csr_matrix(a)
        a.sort_indices()
        self.n = int(a.shape[0])
        if a.shape != (self.n, self.n):
            raise ValueError("matrix must be square")
        self._rp = np.ascontiguousarray(a.indptr, np.int64)
        self._ci = np.ascontiguousarray(a.indices, np.int32)
        self._va = np.ascontiguousarray(a.data, np.float64)
        lib = nat.lib()
        h = C.c_void_p()
        rc = lib.h2b_cg_create(self.n, self._rp.ctypes.data_as(C.POINTER(C.c_int64)),
                               self._ci.ctypes.data_as(C.POINTER(C.c_int32)),
                               self._va.ctypes.data_as(C.POINTER(C.c_double)), C.byref(h))
        if rc == nat.H2B_EINVAL:
            raise ValueError(lib.h2b_last_error().decode())
        nat.check(rc, "h2b_cg_create")
        self._h = h
        self._lib = lib

    def solve(self, b, tol: float = 1e-10, max_iter: int | None = None, deflate_constants: bool = False):
        n = self.n
        if max_iter is None:
            max_iter = 10 * n
        b = np.ascontiguousarray(b, dtype=np.float64)
        if b.shape != (n,):
            raise ValueError(f"rhs must have shape ({n},)")
        if np.linalg.norm(b) == 0.0:
            return np.zeros(n), SolveReport(0, 0.0, True)
        if deflate_constants and abs(b.sum()) > 1e-10 * np.abs(b).sum():  # solver.py:68-70
            raise ValueError("incompatible rhs: not orthogonal to the constant kernel")
        x = np.empty(n)
        it = C.c_int64(0)
        res = C.c_double(0.0)
        rc = self._lib.h2b_cg_solve(self._h, nat.as_d_ptr(b), nat.as_d_ptr(x), float(tol),
                                    int(bool(deflate_constants)), int(max_iter), C.byref(it), C.byref(res))
        if rc == nat.H2B_ECONV:
            raise ConvergenceError(self._lib.h2b_last_error().decode())
        nat.check(rc, "h2b_cg_solve")
        return x, SolveReport(int(it.value), float(res.value), float(res.value) <= tol)

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.h2b_cg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def cg_solve(a, b, tol: float = 1e-10, max_iter: int | None = None, deflate_constants: bool = False):
    """solver.py:44-98 with precond=jacobi_preconditioner(a), on the GPU."""
    solver = GpuCG(a)
    try:
        return solver.solve(b, tol=tol, max_iter=max_iter, deflate_constants=deflate_constants)
    finally:
        solver.close()


def tet_gradients(mesh):
    """fem.py:32-50: per-tet volumes and P1 gradients."""
    p = mesh.nodes[mesh.tets]
    vols = np.einsum("ij,ij->i", p[:, 1] - p[:, 0], np.cross(p[:, 2] - p[:, 0], p[:, 3] - p[:, 0])) / 6.0
    bad = np.flatnonzero(vols <= 0.0)
    if bad.size:
        raise ValueError(f"tetrahedron {int(bad[0])} is degenerate (volume {vols[bad[0]]:g})")
    jac = np.stack([p[:, 1] - p[:, 0], p[:, 2] - p[:, 0], p[:, 3] - p[:, 0]], axis=1)
    inv = np.linalg.inv(jac)
    grads = np.empty((vols.shape[0], 4, 3))
    grads[:, 1:] = np.swapaxes(inv, 1, 2)
    grads[:, 0] = -grads[:, 1:].sum(axis=1)
    return vols, grads


def assemble_stiffness(mesh) -> csr_matrix:
    """fem.py:53-62."""
    vols, grads = tet_gradients(mesh)
    ke = np.einsum("t,tid,tjd->tij", vols, grads, grads)
    rows = np.repeat(mesh.tets, 4, axis=1).reshape(-1)
    cols = np.tile(mesh.tets, (1, 4)).reshape(-1)
    n = mesh.n_nodes
    return coo_matrix((ke.reshape(-1), (rows, cols)), shape=(n, n)).tocsr()


def assemble_u1_rhs(mesh, m_nodal: np.ndarray) -> np.ndarray:
    """fem.py:65-76."""
    if m_nodal.shape != (mesh.n_nodes, 3):
        raise ValueError(f"magnetization must have shape ({mesh.n_nodes}, 3)")
    vols, grads = tet_gradients(mesh)
    m_bar = m_nodal[mesh.tets].mean(axis=1)
    contrib = np.einsum("t,td,tid->ti", vols, m_bar, grads)
    b = np.zeros(mesh.n_nodes)
    np.add.at(b, mesh.tets.reshape(-1), contrib.reshape(-1))
    return b


def solve_u1(mesh, m_nodal, tol: float = 1e-10, max_iter: int | None = None, stiffness=None):
    """fem.py:79-95: the zero-mean Neumann potential, deflated CG on the GPU."""
    a = assemble_stiffness(mesh) if stiffness is None else stiffness
    b = assemble_u1_rhs(mesh, m_nodal)
    if np.linalg.norm(b) == 0.0:
        return np.zeros(mesh.n_nodes), SolveReport(0, 0.0, True)
    return cg_solve(a, b, tol=tol, max_iter=max_iter, deflate_constants=True)


def solve_u2(mesh, dirichlet, tol: float = 1e-10, max_iter: int | None = None, stiffness=None):
    """fem.py:98-121: the Laplace problem on the interior block, CG on the GPU."""
    dirichlet = np.asarray(dirichlet, dtype=np.float64)
    if dirichlet.shape != (mesh.n_boundary,):
        raise ValueError(f"dirichlet data must have shape ({mesh.n_boundary},)")
    a = assemble_stiffness(mesh) if stiffness is None else stiffness
    u = np.zeros(mesh.n_nodes)
    u[mesh.boundary_nodes] = dirichlet
    interior = np.setdiff1d(np.arange(mesh.n_nodes), mesh.boundary_nodes)
    if interior.size == 0:
        return u, SolveReport(0, 0.0, True)
    a_ii = a[interior][:, interior].tocsr()
    rhs = -(a[interior] @ u)
    x, report = cg_solve(a_ii, rhs, tol=tol, max_iter=max_iter)
    u[interior] = x
    return u, report


def compute_field(mesh, u: np.ndarray) -> np.ndarray:
    """fem.py:124-130: H = -grad u per tet."""
    if u.shape != (mesh.n_nodes,):
        raise ValueError(f"potential must have shape ({mesh.n_nodes},)")
    _, grads = tet_gradients(mesh)
    return -np.einsum("ti,tid->td", u[mesh.tets], grads)


def magnetostatic_energy(mesh, m_nodal: np.ndarray, h_tet: np.ndarray):
    """fem.py:133-146: e_d = -1/2 <M . H> and e_d / K_d."""
    nt = mesh.tets.shape[0]
    if h_tet.shape != (nt, 3):
        raise ValueError(f"field must have shape ({nt}, 3)")
    vols, _ = tet_gradients(mesh)
    m_bar = m_nodal[mesh.tets].mean(axis=1)
    energy = -0.5 * np.einsum("t,td,td->", vols, m_bar, h_tet)
    e_d = energy / vols.sum()
    return e_d, e_d / STRAY_FIELD_CONSTANT
