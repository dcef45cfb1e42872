"""Restated FEM steps either side of the boundary operator — TEST
INFRASTRUCTURE ONLY.

The uniformly-magnetized-sphere energy check (north_star) runs
the reference pipeline ``compute_demag`` (pipeline.py:46-63) with the GPU
H² product in the middle.  The reference is absent on the GPU box, so its
FEM pieces are restated here:

* P1 gradients / stiffness           fem.py:32-62
* Neumann right-hand side            fem.py:65-76
* deflated Jacobi-PCG                solver.py:27-98
* solve_u1 / solve_u2                fem.py:79-121
* field and energy                   fem.py:124-146
"""

from __future__ import annotations

import numpy as np
from scipy.sparse import coo_matrix

__all__ = ["compute_demag", "DemagResult"]


class DemagResult:
    def __init__(self, **kw):
        self.__dict__.update(kw)


def _gradients(nodes, tets):
    p = nodes[tets]
    vols = np.einsum("ij,ij->i", p[:, 1] - p[:, 0], np.cross(p[:, 2] - p[:, 0], p[:, 3] - p[:, 0])) / 6.0
    jac = np.stack([p[:, 1] - p[:, 0], p[:, 2] - p[:, 0], p[:, 3] - p[:, 0]], axis=1)
    inv = np.linalg.inv(jac)
    g = np.empty((vols.shape[0], 4, 3))
    g[:, 1:] = np.swapaxes(inv, 1, 2)
    g[:, 0] = -g[:, 1:].sum(axis=1)
    return vols, g


def _stiffness(nodes, tets, vols, g):
    ke = np.einsum("t,tid,tjd->tij", vols, g, g)
    rows = np.repeat(tets, 4, axis=1).reshape(-1)
    cols = np.tile(tets, (1, 4)).reshape(-1)
    n = nodes.shape[0]
    return coo_matrix((ke.reshape(-1), (rows, cols)), shape=(n, n)).tocsr()


def _pcg(a, b, tol, deflate):
    n = b.shape[0]
    max_iter = 10 * n
    b = np.asarray(b, dtype=np.float64)
    bn = np.linalg.norm(b)
    if bn == 0.0:
        return np.zeros(n), 0
    inv = 1.0 / np.asarray(a.diagonal(), dtype=np.float64)
    defl = (lambda v: v - v.mean()) if deflate else (lambda v: v)
    if deflate:
        b = defl(b)
    x = np.zeros(n)
    r = b.copy()
    z = defl(inv * r)
    p = z.copy()
    rz = float(r @ z)
    it = 0
    res = np.linalg.norm(r) / bn
    while res > tol and it < max_iter:
        ap = a @ p
        alpha = rz / float(p @ ap)
        x += alpha * p
        r -= alpha * ap
        z = defl(inv * r)
        rz_new = float(r @ z)
        p = z + (rz_new / rz) * p
        rz = rz_new
        it += 1
        res = np.linalg.norm(r) / bn
    if deflate:
        x = defl(x)
    return x, it


def stiffness(mesh):
    """P1 stiffness of a tet mesh (fem.py:51-62)."""
    vols, g = _gradients(mesh.nodes, mesh.tets)
    return _stiffness(mesh.nodes, mesh.tets, vols, g)


def rhs_u1(mesh, m_nodal):
    """Neumann right-hand side of u1 (fem.py:65-76)."""
    vols, g = _gradients(mesh.nodes, mesh.tets)
    m_bar = m_nodal[mesh.tets].mean(axis=1)
    contrib = np.einsum("t,td,tid->ti", vols, m_bar, g)
    rhs = np.zeros(mesh.nodes.shape[0])
    np.add.at(rhs, mesh.tets.reshape(-1), contrib.reshape(-1))
    return rhs


def compute_demag(mesh, m_nodal, apply_boundary_operator, tol: float = 1e-10) -> DemagResult:
    """``apply_boundary_operator(u1|boundary) -> u2|boundary`` is the product
    under test (GPU h2_matvec, or the oracle for the CPU self-check)."""
    nodes, tets = mesh.nodes, mesh.tets
    vols, g = _gradients(nodes, tets)
    a = _stiffness(nodes, tets, vols, g)
    m_bar = m_nodal[tets].mean(axis=1)
    contrib = np.einsum("t,td,tid->ti", vols, m_bar, g)
    rhs = np.zeros(nodes.shape[0])
    np.add.at(rhs, tets.reshape(-1), contrib.reshape(-1))
    u1, it1 = _pcg(a, rhs, tol, deflate=True)
    u2_b = apply_boundary_operator(u1[mesh.boundary_nodes])
    u2 = np.zeros(nodes.shape[0])
    u2[mesh.boundary_nodes] = u2_b
    interior = np.setdiff1d(np.arange(nodes.shape[0]), mesh.boundary_nodes)
    a_ii = a[interior][:, interior].tocsr()
    x, it2 = _pcg(a_ii, -(a[interior] @ u2), tol, deflate=False)
    u2[interior] = x
    u = u1 + u2
    h = -np.einsum("ti,tid->td", u[tets], g)
    energy = -0.5 * np.einsum("t,td,td->", vols, m_bar, h)
    e_d = energy / vols.sum()
    return DemagResult(u1=u1, u2=u2, u2_boundary=u2_b, e_d=e_d, e_d_over_kd=e_d / 0.5,
                       u1_iterations=it1, u2_iterations=it2)
