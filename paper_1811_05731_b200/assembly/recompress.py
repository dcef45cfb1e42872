"""H -> H² recompression (restates hmatrix/h2.py:86-183).

For every cluster, the factors of all admissible blocks anchored at the
cluster or at one of its ancestors (weighted by the R factor of the opposite
factor's QR) are restricted to the cluster's index range and stacked; a
relative truncated SVD (s > eps_rec * s[0]) gives the basis.  Leaves keep it
explicitly, inner clusters only through the transfer matrices of their
children (the basis is orthonormal and nested).  Coupling matrices are
S_b = (V_t^T A_b)(B_b^T W_s) with the explicit bases.
"""

from __future__ import annotations

import numpy as np

from ..h2 import H2Matrix

__all__ = ["recompress", "basis_side"]


def _truncated_basis(z: np.ndarray, eps: float) -> np.ndarray:
    if z.shape[1] == 0:
        return np.zeros((z.shape[0], 0))
    u, s, _ = np.linalg.svd(z, full_matrices=False)
    if s.size == 0 or s[0] == 0.0:
        return np.zeros((z.shape[0], 0))
    return u[:, : int(np.sum(s > eps * s[0]))]


def basis_side(tree, anchored: dict, eps: float):
    """One side of the nested basis.  ``anchored[cid]`` lists (factor,
    weight) of the blocks whose cluster on this side is ``cid``."""
    basis, transfer, explicit = {}, {}, {}

    def visit(c, inherited):
        mine = [(f @ w.T, c.start) for f, w in anchored.get(c.cid, ())]
        current = inherited + mine
        pieces = [m[c.start - s0: c.end - s0] for m, s0 in current]
        if c.is_leaf:
            v = _truncated_basis(np.hstack(pieces) if pieces else np.zeros((c.size, 0)), eps)
            basis[c.cid] = v
            explicit[c.cid] = v
            return v
        kids = [visit(ch, current) for ch in c.children]
        if pieces:
            z = np.hstack(pieces)
            proj, off = [], 0
            for ch, v in zip(c.children, kids):
                proj.append(v.T @ z[off: off + ch.size])
                off += ch.size
            vhat = _truncated_basis(np.vstack(proj), eps)
        else:
            vhat = np.zeros((sum(v.shape[1] for v in kids), 0))
        parts, off = [], 0
        for ch, v in zip(c.children, kids):
            e = vhat[off: off + v.shape[1]]
            transfer[ch.cid] = e
            parts.append(v @ e)
            off += v.shape[1]
        full = np.vstack(parts)
        explicit[c.cid] = full
        return full

    visit(tree.root, [])
    return basis, transfer, explicit


def recompress(tree, n: int, lowrank: list, dense: list, eps_rec: float, workers: int = 1) -> H2Matrix:
    """``lowrank``: (row cid, col cid, A, B) with block = A @ B.T, in leaf-
    block order; ``dense``: (row cid, col cid, matrix)."""
    if eps_rec < 0.0:
        raise ValueError("epsilon_rec must be >= 0")
    rows: dict = {}
    cols: dict = {}
    for t, s, a, b in lowrank:
        if a.shape[1] == 0:
            continue
        _, rb = np.linalg.qr(b)
        _, ra = np.linalg.qr(a)
        rows.setdefault(t, []).append((a, rb))
        cols.setdefault(s, []).append((b, ra))
    rbasis, rtrans, rexp = basis_side(tree, rows, eps_rec)
    cbasis, ctrans, cexp = basis_side(tree, cols, eps_rec)
    op = H2Matrix(tree=tree, n=n, row_basis=rbasis, row_transfer=rtrans,
                  col_basis=cbasis, col_transfer=ctrans)
    for t, s, a, b in lowrank:
        op.coupling.append((t, s, (rexp[t].T @ a) @ (b.T @ cexp[s])))
    for t, s, m in dense:
        op.near.append((t, s, m))
    return op
