"""H -> H² recompression (restates hmatrix/h2.py:86-183).

For every cluster, the factors of all admissible blocks anchored at the
cluster or at one of its ancestors (weighted by the R factor of the opposite
factor's QR) are restricted to the cluster's index range and stacked; a
relative truncated SVD (s > eps_rec * s[0]) gives the basis.  Leaves keep it
explicitly, inner clusters only through the transfer matrices of their
children (the basis is orthonormal and nested).  Coupling matrices are
S_b = (V_t^T A_b)(B_b^T W_s) with the explicit bases.

Parallelism (threads: the work is LAPACK/BLAS calls that release the GIL,
one BLAS thread each): the per-block QR factors and products, the subtrees
below a split depth, and the coupling products run concurrently.  The
top-down inherited lists are built first and the subtrees' results are
combined bottom-up with the serial code, so the result is identical to the
serial recursion operation for operation.
"""

from __future__ import annotations

import os
import time
from concurrent.futures import ThreadPoolExecutor

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


def _truncated_basis_gram(z: np.ndarray, eps: float) -> np.ndarray:
    """The same subspace from the Gram matrix z z^T (rows <= ~100, columns
    up to thousands): eigenvalues are the squared singular values, so the
    cut s > eps * s0 is lambda > eps^2 * lambda0.  Used for large operators
    (fast build); equal to the SVD's basis up to rounding and column signs."""
    if z.shape[1] == 0 or z.shape[0] == 0:
        return np.zeros((z.shape[0], 0))
    lam, v = np.linalg.eigh(z @ z.T)
    lam, v = lam[::-1], v[:, ::-1]
    if lam[0] <= 0.0:
        return np.zeros((z.shape[0], 0))
    keep = int(np.sum(np.sqrt(np.maximum(lam, 0.0)) > eps * np.sqrt(lam[0])))
    return np.ascontiguousarray(v[:, :keep])


class _Side:
    def __init__(self, eps, fast=False):
        self.eps = eps
        self.tb = _truncated_basis_gram if fast else _truncated_basis
        self.basis, self.transfer, self.explicit = {}, {}, {}
        self.t_leaf = self.t_inner = 0.0  # summed over threads (diagnostics)

    def combine(self, c, current, kids):
        """Inner cluster: projection of the stacked restricted factors onto
        the children's bases, truncated; children's transfers."""
        t0 = time.perf_counter()
        full = self._combine(c, current, kids)
        self.t_inner += time.perf_counter() - t0
        return full

    def _combine(self, c, current, kids):
        pieces = [_restrict(e, c) for e in current]
        if pieces:
            z = np.hstack(pieces)
            proj, off = [], 0
            for ch, v in zip(c.children, kids):
                proj.append(v.T @ z[off: off + ch.size])
                off += ch.size
            vhat = self.tb(np.vstack(proj), self.eps)
        else:
            vhat = np.zeros((sum(v.shape[1] for v in kids), 0))
        parts, off = [], 0
        for ch, v in zip(c.children, kids):
            e = vhat[off: off + v.shape[1]]
            self.transfer[ch.cid] = e
            parts.append(v @ e)
            off += v.shape[1]
        full = np.vstack(parts)
        self.explicit[c.cid] = full
        return full

    def visit(self, c, inherited, own):
        current = inherited + own.get(c.cid, [])
        if c.is_leaf:
            t0 = time.perf_counter()
            pieces = [_restrict(e, c) for e in current]
            v = self.tb(np.hstack(pieces) if pieces else np.zeros((c.size, 0)), self.eps)
            self.t_leaf += time.perf_counter() - t0
            self.basis[c.cid] = v
            self.explicit[c.cid] = v
            return v
        kids = [self.visit(ch, current, own) for ch in c.children]
        return self.combine(c, current, kids)


def _weighted(f: np.ndarray, w) -> np.ndarray:
    """f @ w.T for a weight given as a matrix, a diagonal (1-D array) or the
    identity (None) -- the batched HCA's factors have orthonormal B and
    A^T A = S^2, so their weights are I and diag(s) and need no k x k
    matrices (37 GB of them on the 1M-node disk)."""
    if w is None:
        return f
    if w.ndim == 1:
        return f * w[None, :]
    return f @ w.T


def _restrict(entry, c):
    """Rows of cluster c of an anchored, weighted factor.  Entries are
    (weighted factor, anchor start) or, for a diagonal weight, (factor,
    anchor start, weight): the weight is applied to the restricted rows
    only (elementwise, so the same numbers as weighting first), instead of
    holding a weighted copy of every factor (half the factor memory)."""
    m, s0 = entry[0], entry[1]
    r = m[c.start - s0: c.end - s0]
    return r * entry[2][None, :] if len(entry) == 3 else r


def basis_side(tree, anchored: dict, eps: float, pool=None, split_depth: int = 0, fast: bool = False):
    """One side of the nested basis.  ``anchored[cid]`` lists (factor,
    weight) of the blocks whose cluster on this side is ``cid``."""
    side = _Side(eps, fast)
    t_start = time.perf_counter()
    items = [(cid, f, w) for cid, lst in anchored.items() for f, w in lst]
    full = [i for i, (_, f, w) in enumerate(items) if w is not None and w.ndim != 1]
    mats = dict(zip(full, pool.map(lambda i: _weighted(items[i][1], items[i][2]), full) if pool
                    else [_weighted(items[i][1], items[i][2]) for i in full]))
    own: dict = {}
    for i, (cid, f, w) in enumerate(items):
        s0 = tree.clusters[cid].start
        if i in mats:
            own.setdefault(cid, []).append((mats[i], s0))
        elif w is None:
            own.setdefault(cid, []).append((f, s0))
        else:
            own.setdefault(cid, []).append((f, s0, w))
    basis_side.last = {"weighting": time.perf_counter() - t_start}
    if pool is None or split_depth <= 0:
        side.visit(tree.root, [], own)
        basis_side.last.update(leaf_cpu=side.t_leaf, inner_cpu=side.t_inner)
        return side.basis, side.transfer, side.explicit
    # top-down: inherited lists down to the split depth
    frontier, top = [(tree.root, [])], []
    for _ in range(split_depth):
        nxt = []
        for c, inh in frontier:
            if c.is_leaf:
                nxt.append((c, inh))
                continue
            cur = inh + own.get(c.cid, [])
            top.append((c, cur))
            nxt.extend((ch, cur) for ch in c.children)
        frontier = nxt
    # subtrees in parallel (each writes its own clusters' entries)
    list(pool.map(lambda ci: side.visit(ci[0], ci[1], own), frontier))
    # bottom-up over the top part, children before parents
    for c, cur in reversed(top):
        side.combine(c, cur, [side.explicit[ch.cid] for ch in c.children])
    basis_side.last.update(leaf_cpu=side.t_leaf, inner_cpu=side.t_inner)
    return side.basis, side.transfer, side.explicit


def recompress(tree, n: int, lowrank: list, dense: list, eps_rec: float, workers: int = 1,
               weights: list | None = None, timings: dict | None = None) -> H2Matrix:
    """``lowrank``: (row cid, col cid, A, B) with block = A @ B.T, in leaf-
    block order; ``dense``: (row cid, col cid, matrix).

    ``weights`` (fast build of large operators): per low-rank block the
    pair (W_b, W_a) with W^T W = B^T B and A^T A, replacing the QR R factors
    (only R^T R enters the bases); bases then come from Gram matrices.  A
    weight may be a matrix, a 1-D diagonal or None (identity)."""
    if eps_rec < 0.0:
        raise ValueError("epsilon_rec must be >= 0")
    pool = None
    limiter = None
    if workers > 1:
        try:
            from threadpoolctl import threadpool_limits
            limiter = threadpool_limits(1)
        except Exception:
            limiter = None
        pool = ThreadPoolExecutor(max_workers=workers)
    try:
        fast = weights is not None
        keep_ids = [i for i, (t, s, a, b) in enumerate(lowrank) if a.shape[1] > 0]
        nz = [lowrank[i] for i in keep_ids]

        def qr_r(t):
            _, _, a, b = t
            return np.linalg.qr(b)[1], np.linalg.qr(a)[1]

        if fast:
            rs = [weights[i] for i in keep_ids]
        else:
            rs = list(pool.map(qr_r, nz)) if pool else [qr_r(t) for t in nz]
        rows: dict = {}
        cols: dict = {}
        for (t, s, a, b), (rb, ra) in zip(nz, rs):
            rows.setdefault(t, []).append((a, rb))
            cols.setdefault(s, []).append((b, ra))
        depth = max(1, int(np.ceil(np.log2(max(2, 4 * workers))))) if pool else 0
        t0 = time.perf_counter()
        rbasis, rtrans, rexp = basis_side(tree, rows, eps_rec, pool, depth, fast)
        t1 = time.perf_counter()
        cbasis, ctrans, cexp = basis_side(tree, cols, eps_rec, pool, depth, fast)
        t2 = time.perf_counter()
        if timings is not None:
            timings.update(rec_rows=t1 - t0, rec_cols=t2 - t1,
                           **{f"rec_cols_{k}": v for k, v in getattr(basis_side, "last", {}).items()})
        op = H2Matrix(tree=tree, n=n, row_basis=rbasis, row_transfer=rtrans,
                      col_basis=cbasis, col_transfer=ctrans)

        def coupling(blk):
            t, s, a, b = blk
            return (t, s, (rexp[t].T @ a) @ (b.T @ cexp[s]))

        op.coupling.extend(pool.map(coupling, lowrank) if pool else map(coupling, lowrank))
        if timings is not None:
            timings.update(rec_coupling=time.perf_counter() - t2)
        for t, s, m in dense:
            op.near.append((t, s, m))
        return op
    finally:
        if pool is not None:
            pool.shutdown()
        if limiter is not None:
            try:
                limiter.restore_original_limits()
            except Exception:
                pass
