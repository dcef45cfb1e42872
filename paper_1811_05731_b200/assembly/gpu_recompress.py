"""H -> H² recompression on the GPU (hmatrix/h2.py:86-183).

The reference's ``_basis_side`` stacks, for every cluster, the factors of all
admissible blocks anchored at the cluster or an ancestor, restricted to the
cluster's rows, projects the stack onto the children's explicit bases and
takes a truncated SVD.  ``recompress.py`` restates that on host threads (with
Gram matrices for the large workloads).  Here the same bases come out of a
bottom-up sweep over the tree levels that never forms an explicit basis of an
inner cluster and reads every factor once:

* the own factors of a cluster t (all |t| x k_b, anchored at t) are packed
  side by side into one row-major |t| x C_t block; the columns a cluster c
  sees are those of its ancestors' blocks followed by its own
  (``inherited + own``, h2.py:118), so a parent's columns are a *prefix* of
  its children's;
* leaves: G = sum_a R_a diag(w_a^2) R_a^T over the chain of ancestors a, R_a
  the leaf's rows of a's block (``h2b_rc_leaf_gram``); eigenvectors by a
  batched Jacobi solver, one CTA per matrix (``h2b_rc_eigh``); the cut
  s > eps s_0 is lambda > eps^2 lambda_0; the *projected factors*
  P_c = V_c^T R diag(w) (k_c x C_c, column-major) are kept
  (``h2b_rc_leaf_project``);
* inner clusters: the projection of the stacked factors onto the children's
  bases is the stack of the children's P (their first C_c columns -- the
  bases are nested, V_c = blockdiag(V_ch) E), so G = Z Z^T with
  Z = [P_ch1; P_ch2] (``h2b_rc_inner_gram``), the transfers are the rows of
  the eigenvectors and P_c = Vhat^T Z (``h2b_rc_inner_project``);
* coupling matrices S_b = (V_t^T A_b)(B_b^T W_s) (h2.py:171-176) are products
  of the clusters' own columns of P with the weights divided out
  (``h2b_rc_extract_own``, ``h2b_rc_coupling``).

Weights follow recompress.py: a block enters the row side as A_b R_B^T and the
column side as B_b R_A^T (only R^T R matters); the batched HCA's factors have
orthonormal B and orthogonal A columns, so the weights are the identity and
diag(|a_j|).  Blocks that came from the ACA fallback are brought to that form
first (QR of B, SVD of A R_B^T).

Everything is deterministic (no atomics).  The summation order differs from
the host path's, so a kept rank can differ right at the threshold; the
resulting operator approximates the same matrix to the same eps_rec.

The numerical steps go through an ``ops`` object: ``CudaOps`` (libh2b.so, the
product) or, in the CPU tests only, ``oracle/rc_ops_ref.py::NumpyOps``.
"""

from __future__ import annotations

import ctypes as C
import os
import time

import numpy as np

from ..h2 import H2Matrix

__all__ = ["recompress_gpu", "CudaOps", "normalise_block"]

LEAF_MAX = 64     # rows of a leaf the Gram kernel takes
INNER_MAX = 128   # stacked child ranks the inner kernels take


def normalise_block(a: np.ndarray, b: np.ndarray):
    """(a, b) -> (a', b') with a' b'^T = a b^T, b' orthonormal columns and a'
    orthogonal columns (the form of the batched HCA's factors)."""
    if a.shape[1] == 0:
        return a, b
    qb, rb = np.linalg.qr(b)
    u, s, vt = np.linalg.svd(a @ rb.T, full_matrices=False)
    return np.ascontiguousarray(u * s[None, :]), np.ascontiguousarray(qb @ vt.T)


class _Tree:
    """Flat tree arrays: preorder ids, binary inner clusters."""

    def __init__(self, tree):
        cl = tree.clusters
        nc = len(cl)
        self.nc = nc
        self.start = np.array([c.start for c in cl], np.int64)
        self.end = np.array([c.end for c in cl], np.int64)
        self.child = np.full((nc, 2), -1, np.int64)
        self.parent = np.full(nc, -1, np.int64)
        for c in cl:
            if c.children:
                if len(c.children) != 2:
                    raise ValueError("recompress_gpu needs a binary cluster tree")
                for j, ch in enumerate(c.children):
                    self.child[c.cid, j] = ch.cid
                    self.parent[ch.cid] = c.cid
        self.depth = np.zeros(nc, np.int64)
        # parents need not precede children in cid order: walk from the root
        root = tree.root.cid
        stack = [root]
        topo = []
        while stack:
            c = stack.pop()
            topo.append(c)
            for ch in self.child[c]:
                if ch >= 0:
                    self.depth[ch] = self.depth[c] + 1
                    stack.append(int(ch))
        self.topo = np.array(topo, np.int64)
        self.maxdepth = int(self.depth.max())
        # ancestors root -> c, padded with -1
        self.anc = np.full((nc, self.maxdepth + 1), -1, np.int32)
        for c in topo:
            d = self.depth[c]
            if d > 0:
                self.anc[c, :d] = self.anc[self.parent[c], :d]
            self.anc[c, d] = c
        self.is_leaf = self.child[:, 0] < 0


class _SidePlan:
    """Column bookkeeping of one side: which blocks a cluster owns and where
    their columns sit."""

    def __init__(self, T: _Tree, cid: np.ndarray, kb: np.ndarray):
        nc = T.nc
        order = np.argsort(cid, kind="stable")  # own blocks in lowrank order per cluster
        self.order = order
        self.cown = np.bincount(cid, weights=kb, minlength=nc).astype(np.int64)
        # column start of a block inside its cluster's own block
        csum = np.cumsum(kb[order]) - kb[order]
        first = np.zeros(nc + 1, np.int64)
        np.cumsum(np.bincount(cid, minlength=nc), out=first[1:])
        base = np.zeros(order.size, np.int64)
        nz = first[:-1] < first[1:]
        base_per_cluster = np.zeros(nc, np.int64)
        base_per_cluster[nz] = csum[first[:-1][nz]]
        base = csum - base_per_cluster[cid[order]]
        self.colstart = np.zeros(cid.size, np.int64)
        self.colstart[order] = base
        self.first = first  # blocks of cluster c: order[first[c]:first[c+1]]
        self.ccur = np.zeros(nc, np.int64)
        for c in T.topo:
            p = T.parent[c]
            self.ccur[c] = (self.ccur[p] if p >= 0 else 0) + self.cown[c]
        size = T.end - T.start
        self.foff = np.zeros(nc + 1, np.int64)
        np.cumsum(size * self.cown, out=self.foff[1:])
        self.woff = np.zeros(nc + 1, np.int64)
        np.cumsum(self.cown, out=self.woff[1:])


class CudaOps:
    """The recompression kernels of libh2b.so (csrc/recompress.cu) on torch
    device memory.  No fallback: raises without the library or a GPU."""

    def __init__(self, device: str = "cuda"):
        import torch
        from .. import _native as nat
        if not torch.cuda.is_available():
            raise RuntimeError("recompress_gpu needs a CUDA device (there is no CPU fallback)")
        self.torch, self.nat, self.lib = torch, nat, nat.lib()
        self.dev = torch.device(device)
        vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int32
        sig = {  # without the trailing stream argument
            "h2b_rc_leaf_gram": [i64] + [vp] * 7 + [i32, vp, vp, vp, i32, vp],
            "h2b_rc_eigh": [i64, vp, vp, i32, vp, i32],
            "h2b_rc_leaf_project": [i64] + [vp] * 7 + [i32, vp, vp, vp, vp, i32, vp, vp, vp, vp],
            "h2b_rc_inner_gram": [i64] + [vp] * 6 + [vp, i32],
            "h2b_rc_inner_project": [i64] + [vp] * 6 + [vp, i32, vp, vp],
            "h2b_rc_extract_own": [i64] + [vp] * 11,
            "h2b_rc_coupling": [i64] + [vp] * 13,
        }
        for nm, args in sig.items():
            f = getattr(self.lib, nm)
            f.argtypes = args + [vp]
            f.restype = C.c_int

    # -- memory
    def empty(self, n, dtype=np.float64):
        t = self.torch
        return t.empty(int(max(1, n)), dtype={np.float64: t.float64, np.int64: t.int64, np.int32: t.int32}[dtype],
                       device=self.dev)

    def zeros(self, n, dtype=np.float64):
        a = self.empty(n, dtype)
        a.zero_()
        return a

    def to_device(self, a: np.ndarray):
        t = self.torch
        if a.size == 0:
            return self.empty(1, a.dtype.type)
        return t.from_numpy(np.ascontiguousarray(a)).to(self.dev)

    def to_host(self, a, n=None) -> np.ndarray:
        return (a if n is None else a[:int(n)]).cpu().numpy()

    def upload_into(self, dst, off: int, src: np.ndarray):
        dst[off:off + src.size].copy_(self.torch.from_numpy(src), non_blocking=False)

    def staging(self, n):
        return self.torch.empty(int(n), dtype=self.torch.float64, pin_memory=True).numpy()

    def sync(self):
        self.torch.cuda.synchronize()

    def release(self):
        """Return the caching allocator's blocks to the driver (h2b_create
        allocates the operator with cudaMalloc, outside torch)."""
        self.torch.cuda.synchronize()
        self.torch.cuda.empty_cache()

    def _call(self, name, *args):
        st = self.torch.cuda.current_stream().cuda_stream
        conv = [a.data_ptr() if hasattr(a, "data_ptr") else a for a in args]
        self.nat.check(getattr(self.lib, name)(*conv, st), name)

    # -- kernels (argument meaning: include/h2b.h)
    def leaf_gram(self, ids, start, end, anc, depth, foff, cown, woff, nanc, fac, wts, G, ldg):
        self._call("h2b_rc_leaf_gram", ids.numel(), ids, start, end, anc, depth, foff, cown, nanc, woff, fac, wts,
                   ldg, G)

    def eigh(self, nmat, nvec, G, ldg, lam, sweeps):
        self._call("h2b_rc_eigh", nmat, nvec, G, ldg, lam, sweeps)

    def leaf_project(self, ids, start, end, anc, depth, foff, cown, woff, nanc, fac, wts, V, ldg, k, P, poff, ccur):
        self._call("h2b_rc_leaf_project", ids.numel(), ids, start, end, anc, depth, foff, cown, nanc, woff, fac, wts,
                   V, ldg, k, P, poff, ccur)

    def inner_gram(self, ids, child, k, ccur, Pc, poffc, G, ldg):
        self._call("h2b_rc_inner_gram", ids.numel(), ids, child, k, ccur, Pc, poffc, G, ldg)

    def inner_project(self, ids, child, k, ccur, Pc, poffc, V, ldg, P, poff):
        self._call("h2b_rc_inner_project", ids.numel(), ids, child, k, ccur, Pc, poffc, V, ldg, P, poff)

    def extract_own(self, ids, parent, k, ccur, cown, woff, wts, P, poff, Q, qoff):
        self._call("h2b_rc_extract_own", ids.numel(), ids, parent, k, ccur, cown, woff, wts, P, poff, Q, qoff)

    def coupling(self, nb, bt, bs, rcol, ccol, kb, Qr, qoffr, kr, Qc, qoffc, kc, S, soff):
        self._call("h2b_rc_coupling", nb, bt, bs, rcol, ccol, kb, Qr, qoffr, kr, Qc, qoffc, kc, S, soff)


def _pack_side(ops, T: _Tree, sp: _SidePlan, cid, factors, weights, say, workers: int = 8):
    """Upload the side's factors: per cluster its own blocks side by side
    (row-major |c| x cown[c]), through a pinned staging buffer filled by a
    few host threads (numpy's copy loops release the GIL)."""
    from concurrent.futures import ThreadPoolExecutor
    total = int(sp.foff[-1])
    fac = ops.empty(total)
    wts = np.ones(max(1, int(sp.woff[-1])))
    stage_n = int(os.environ.get("H2B_RC_STAGE_DOUBLES", 1 << 26))  # 512 MB of doubles
    stage = ops.staging(min(max(total, 1), stage_n))
    size = T.end - T.start
    owners = np.flatnonzero(sp.cown > 0)

    def fill_one(c, base):
        """Cluster c's packed block into stage[foff[c] - base ...], and its weights."""
        blocks = sp.order[sp.first[c]:sp.first[c + 1]]
        o = int(sp.foff[c]) - base
        np.concatenate([factors[b] for b in blocks], axis=1,
                       out=stage[o:o + int(size[c] * sp.cown[c])].reshape(int(size[c]), int(sp.cown[c])))
        if weights is not None:
            w0 = int(sp.woff[c])
            for b in blocks:
                kb = factors[b].shape[1]
                wts[w0:w0 + kb] = weights[b]
                w0 += kb

    with ThreadPoolExecutor(max_workers=max(1, workers)) as pool:
        i = 0
        while i < owners.size:
            c0 = int(owners[i])
            base = int(sp.foff[c0])
            need0 = int(size[c0] * sp.cown[c0])
            if need0 > stage.size:  # a block larger than the staging buffer goes on its own
                blocks = sp.order[sp.first[c0]:sp.first[c0 + 1]]
                big = np.concatenate([factors[b] for b in blocks], axis=1)
                ops.upload_into(fac, base, big.ravel())
                if weights is not None:
                    wts[int(sp.woff[c0]):int(sp.woff[c0 + 1])] = np.concatenate([weights[b] for b in blocks])
                i += 1
                continue
            # the clusters that fit the staging buffer together (foff is contiguous in cluster order)
            j = int(np.searchsorted(sp.foff[owners + 1], base + stage.size, side="right"))
            j = max(j, i + 1)
            batch = owners[i:j]
            list(pool.map(lambda c: fill_one(int(c), base), batch, chunksize=max(1, batch.size // (8 * max(1, workers)))))
            fill = int(sp.foff[int(batch[-1]) + 1]) - base
            ops.upload_into(fac, base, stage[:fill])
            i = j
    return fac, ops.to_device(wts)


def _basis_side(ops, T: _Tree, sp: _SidePlan, fac, wts, eps, n_jacobi_sweeps=30):
    """Bottom-up over the depths.  Returns (k, basis, transfer, Q, qoff):
    ranks, leaf bases {cid: |c| x k}, transfers {cid: k_c x k_parent}, and the
    own columns of the projected factors (device array + offsets)."""
    nc = T.nc
    k = np.zeros(nc, np.int64)
    basis, transfer = {}, {}
    d_start, d_end = ops.to_device(T.start), ops.to_device(T.end)
    d_anc, d_depth = ops.to_device(T.anc.ravel()), ops.to_device(T.depth)
    d_foff, d_cown, d_woff = ops.to_device(sp.foff), ops.to_device(sp.cown), ops.to_device(sp.woff)
    d_ccur, d_child, d_parent = ops.to_device(sp.ccur), ops.to_device(T.child.ravel()), ops.to_device(T.parent)
    nanc = T.maxdepth + 1
    size = T.end - T.start
    # own columns of P, with the weights divided out: k_c x cown[c], column-major
    qoff = np.zeros(nc + 1, np.int64)
    Q_parts = {}
    prevP = prev_poff = None
    d_k = ops.zeros(nc, np.int64)
    for d in range(T.maxdepth, -1, -1):
        at = np.flatnonzero(T.depth == d)
        leaves = at[T.is_leaf[at]]
        inner = at[~T.is_leaf[at]]
        if leaves.size and size[leaves].max() > LEAF_MAX:
            raise NotImplementedError(f"recompress_gpu: leaves of more than {LEAF_MAX} rows")
        m_in = (k[T.child[inner, 0]] + k[T.child[inner, 1]]) if inner.size else np.zeros(0, np.int64)
        if inner.size and m_in.max() > INNER_MAX:
            raise NotImplementedError(f"recompress_gpu: stacked child ranks above {INNER_MAX}")
        # --- Gram matrices of the level: leaves first, then inner clusters
        ids = np.concatenate([leaves, inner])
        nvec = np.concatenate([size[leaves], m_in]).astype(np.int64)
        nmat = ids.size
        ldg = int(max(1, nvec.max() if nmat else 1))
        G = ops.zeros(nmat * ldg * ldg)
        d_ids = ops.to_device(ids)
        if leaves.size:
            ops.leaf_gram(d_ids[:leaves.size], d_start, d_end, d_anc, d_depth, d_foff, d_cown, d_woff, nanc,
                          fac, wts, G, ldg)
        if inner.size:
            ops.inner_gram(d_ids[leaves.size:], d_child, d_k, d_ccur, prevP, prev_poff,
                           G[leaves.size * ldg * ldg:], ldg)
        lam = ops.zeros(nmat * ldg)
        ops.eigh(nmat, ops.to_device(nvec), G, ldg, lam, n_jacobi_sweeps)
        lam_h = ops.to_host(lam, nmat * ldg).reshape(nmat, ldg)
        # the relative cut (recompress._truncated_basis_gram)
        for i in range(0, nmat, 1 << 16):
            L = lam_h[i:i + (1 << 16)]
            nv = nvec[i:i + (1 << 16)]
            valid = np.arange(ldg)[None, :] < nv[:, None]
            l0 = np.where(nv > 0, L[:, 0], 0.0)
            s = np.sqrt(np.maximum(L, 0.0))
            keep = (s > eps * np.sqrt(np.maximum(l0, 0.0))[:, None]) & valid & (l0 > 0.0)[:, None]
            k[ids[i:i + (1 << 16)]] = keep.sum(axis=1)
        d_k = ops.to_device(k)
        # --- projected factors of the level
        poff = np.zeros(nc + 1, np.int64)
        pc = np.zeros(nc, np.int64)
        pc[ids] = k[ids] * sp.ccur[ids]
        np.cumsum(pc, out=poff[1:])
        P = ops.empty(int(poff[-1]))
        d_poff = ops.to_device(poff)
        if leaves.size:
            ops.leaf_project(d_ids[:leaves.size], d_start, d_end, d_anc, d_depth, d_foff, d_cown, d_woff, nanc,
                             fac, wts, G, ldg, d_k, P, d_poff, d_ccur)
        if inner.size:
            ops.inner_project(d_ids[leaves.size:], d_child, d_k, d_ccur, prevP, prev_poff,
                              G[leaves.size * ldg * ldg:], ldg, P, d_poff)
        # own columns for the coupling matrices
        own = ids[(sp.cown[ids] > 0) & (k[ids] > 0)]
        if own.size:
            qsz = np.zeros(nc, np.int64)
            qsz[own] = k[own] * sp.cown[own]
            qo = np.zeros(nc + 1, np.int64)
            np.cumsum(qsz, out=qo[1:])
            Q = ops.empty(int(qo[-1]))
            ops.extract_own(ops.to_device(own), d_parent, d_k, d_ccur, d_cown, d_woff, wts, P, d_poff, Q,
                            ops.to_device(qo))
            Q_parts[d] = (Q, qo, own)
        # --- results to the host: eigenvectors as bases / transfers
        Vh = ops.to_host(G, nmat * ldg * ldg).reshape(nmat, ldg, ldg)
        for i, c in enumerate(leaves):
            basis[int(c)] = np.ascontiguousarray(Vh[i, :size[c], :k[c]])
        for j, c in enumerate(inner):
            i = leaves.size + j
            c1, c2 = T.child[c]
            v = Vh[i, :m_in[j], :k[c]]
            transfer[int(c1)] = np.ascontiguousarray(v[:k[c1]])
            transfer[int(c2)] = np.ascontiguousarray(v[k[c1]:])
        prevP, prev_poff = P, d_poff
        del G, lam
    return k, basis, transfer, Q_parts


def recompress_gpu(tree, n: int, lowrank: list, dense: list, eps_rec: float, weights: list,
                   ops=None, timings: dict | None = None, log=None) -> H2Matrix:
    """Same contract as ``recompress.recompress(..., weights=...)``."""
    if eps_rec < 0.0:
        raise ValueError("epsilon_rec must be >= 0")
    ops = ops or CudaOps()
    say = log or (lambda *a: None)
    t0 = time.perf_counter()
    T = _Tree(tree)
    nb = len(lowrank)
    bt = np.array([b[0] for b in lowrank], np.int64)
    bs = np.array([b[1] for b in lowrank], np.int64)
    A = [b[2] for b in lowrank]
    B = [b[3] for b in lowrank]
    wcol = [None] * nb
    for i in range(nb):
        wb, wa = weights[i] if weights is not None else (0, 0)
        if A[i].shape[1] == 0:
            wcol[i] = np.zeros(0)
        elif weights is None or wb is not None or wa is None or np.ndim(wa) != 1:
            A[i], B[i] = normalise_block(A[i], B[i])
            wcol[i] = np.linalg.norm(A[i], axis=0)
        else:
            wcol[i] = wa
    kb = np.array([a.shape[1] for a in A], np.int64)
    sides = {}
    for name, cid, fac_list, w in (("rows", bt, A, None), ("cols", bs, B, wcol)):
        t1 = time.perf_counter()
        sp = _SidePlan(T, cid, kb)
        fac, wts = _pack_side(ops, T, sp, cid, fac_list, w, say)
        ops.sync()
        t2 = time.perf_counter()
        k, basis, transfer, Q_parts = _basis_side(ops, T, sp, fac, wts, eps_rec)
        ops.sync()
        t3 = time.perf_counter()
        del fac
        sides[name] = (sp, k, basis, transfer, Q_parts)
        if timings is not None:
            timings[f"rec_{name}_pack"] = t2 - t1
            timings[f"rec_{name}"] = t3 - t2
    spr, kr, rbasis, rtrans, Qr_parts = sides["rows"]
    spc, kc, cbasis, ctrans, Qc_parts = sides["cols"]
    op = H2Matrix(tree=tree, n=n, row_basis=rbasis, row_transfer=rtrans, col_basis=cbasis, col_transfer=ctrans)
    # --- coupling matrices: one flat Q per side, then one launch over the blocks
    t4 = time.perf_counter()

    def flatten(parts, nc):
        tot = sum(int(qo[-1]) for _, qo, _ in parts.values())
        Q = ops.empty(tot)
        qoff = np.zeros(nc, np.int64)
        pos = 0
        for d in sorted(parts):
            q, qo, own = parts[d]
            m = int(qo[-1])
            if m:
                Q[pos:pos + m] = q[:m]
            qoff[own] = qo[own] + pos
            pos += m
        return Q, qoff

    Qr, qoffr = flatten(Qr_parts, T.nc)
    Qc, qoffc = flatten(Qc_parts, T.nc)
    ssz = kr[bt] * kc[bs]
    soff = np.zeros(nb + 1, np.int64)
    np.cumsum(ssz, out=soff[1:])
    S = ops.zeros(int(soff[-1]))
    if nb:
        ops.coupling(nb, ops.to_device(bt), ops.to_device(bs), ops.to_device(spr.colstart), ops.to_device(spc.colstart),
                     ops.to_device(kb), Qr, ops.to_device(qoffr), ops.to_device(kr), Qc, ops.to_device(qoffc),
                     ops.to_device(kc), S, ops.to_device(soff))
    Sh = ops.to_host(S, int(soff[-1]))
    for i in range(nb):
        op.coupling.append((int(bt[i]), int(bs[i]), Sh[soff[i]:soff[i + 1]].reshape(int(kr[bt[i]]), int(kc[bs[i]]))))
    for t, s, m in dense:
        op.near.append((t, s, m))
    del S, Qr, Qc, Qr_parts, Qc_parts, sides
    if hasattr(ops, "release"):
        ops.release()
    if timings is not None:
        timings["rec_coupling"] = time.perf_counter() - t4
        timings["rec_total"] = time.perf_counter() - t0
    return op
