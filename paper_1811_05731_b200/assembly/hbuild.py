"""H² construction: the host-side producer of the matvec's input.

The north star keeps the H² structure "built by the reference on the host".
The reference cannot travel to the GPU box, so this module restates its
construction algorithm (/root/reference/pkg/src/strayfield/hmatrix/):

* cluster tree: median bisection on the longest box axis, stable sort,
  preorder ids                                        cluster.py:62-106
* block tree: admissible iff dist > 0 and max(diam) <= eta*dist; split the
  clusters that still have children; leaf blocks in preorder
                                                      cluster.py:117-157
* admissible blocks: hybrid cross approximation — Chebyshev grids, fully
  pivoted ACA on the Green's-function matrix, A by solving with the cross,
  B from analytic panel rows at the pivots, QR/SVD truncation; ACA
  fallback on an ill-conditioned cross               hca.py:38-105,
                                                      lowrank.py:36-164
* near field: dense collocation blocks of M = K + D  bem.py:221-235
* H -> H²: per-cluster truncated SVD of the agglomerated, QR-weighted block
  rows/columns; transfer matrices; coupling (V^T A)(B^T W)
                                                      h2.py:86-183

The dense linear algebra runs in numpy with the reference's operation order
(on a fork pool); the collocation entries — 72% of the reference's build
time — run on the GPU (csrc/colloc.cu) through the
``h2b_colloc_*`` C ABI.  A different entry evaluator can be injected
(tests use the CPU restatement in oracle/colloc_ref.py).
"""

from __future__ import annotations

import ctypes as C
import math
import os
import time
import warnings
from dataclasses import dataclass

import numpy as np

from .. import _native as nat
from ..cluster import Cluster, ClusterTree
from ..h2 import H2Matrix
from .geometry import Surface, incidence, panel_table

__all__ = ["CompressionConfig", "build_cluster_tree", "leaf_block_list", "chebyshev_points",
           "green_cross", "aca_full", "aca", "truncate_lowrank", "GpuCollocation",
           "assemble_h2", "BuildReport"]

_FOUR_PI = 4.0 * math.pi
_COND_LIMIT = 1e12


@dataclass(frozen=True)
class CompressionConfig:
    """Compression parameters; defaults are the reference code's
    (hmat.py:19-28), which differ from SPEC's."""

    leaf_size: int = 32
    eta: float = 3.0
    cheb_order: int = 5
    eps: float = 1e-5
    eps_rec: float = 2e-4
    method: str = "hca"


# ---------------------------------------------------------------------------
# cluster tree and block partition
# ---------------------------------------------------------------------------

def build_cluster_tree(points: np.ndarray, leaf_size: int = 32) -> ClusterTree:
    points = np.asarray(points, dtype=np.float64)
    if points.ndim != 2 or points.shape[1] != 3 or points.shape[0] < 1:
        raise ValueError("points must have shape (N, 3) with N >= 1")
    if leaf_size < 1:
        raise ValueError("leaf_size must be >= 1")
    perm = np.arange(points.shape[0], dtype=np.int64)

    def split(start: int, end: int) -> Cluster:
        idx = perm[start:end]
        sub = points[idx]
        lo, hi = sub.min(axis=0), sub.max(axis=0)
        node = Cluster(start, end, lo, hi)
        if end - start > leaf_size:
            axis = int(np.argmax(hi - lo))           # lowest axis on ties
            perm[start:end] = idx[np.argsort(sub[:, axis], kind="stable")]
            half = start + (end - start) // 2
            node.children = (split(start, half), split(half, end))
        return node

    root = split(0, points.shape[0])
    order: list[Cluster] = []
    stack = [root]
    while stack:
        c = stack.pop()
        c.cid = len(order)
        order.append(c)
        stack.extend(reversed(c.children))
    return ClusterTree(root=root, perm=perm, clusters=order)


def _norm3(v: np.ndarray) -> float:
    return float(np.linalg.norm(v))


def leaf_block_list(tree: ClusterTree, eta: float):
    """Leaf blocks of the admissibility block tree, in the reference's
    preorder (``leaf_blocks(build_block_tree(...))``), computed level-
    synchronously.  Returns (row cids, col cids, admissible flags)."""
    if eta <= 0.0:
        raise ValueError("eta must be positive")
    cl = tree.clusters
    nc = len(cl)
    lo = np.array([c.bbox_min for c in cl])
    hi = np.array([c.bbox_max for c in cl])
    diam = np.array([_norm3(c.bbox_max - c.bbox_min) for c in cl])
    child = np.full((nc, 2), -1, np.int64)
    for c in cl:
        if c.children:
            child[c.cid] = [c.children[0].cid, c.children[1].cid]
    T = np.zeros(1, np.int64)
    S = np.zeros(1, np.int64)
    key = np.zeros(1, np.int64)
    out_t, out_s, out_adm, out_key, out_depth = [], [], [], [], []
    depth = 0
    while T.size:
        gap = np.maximum(np.maximum(lo[T] - hi[S], lo[S] - hi[T]), 0.0)
        dist = np.sqrt(np.einsum("ij,ij->i", gap, gap))
        dmax = np.maximum(diam[T], diam[S])
        adm = (dist > 0.0) & (dmax <= eta * dist)
        # decisions within rounding of the threshold: recompute exactly as
        # the reference does (per-pair np.linalg.norm, cluster.py:29-31, 110-114)
        close = (dist > 0.0) & (np.abs(dmax - eta * dist) <= 1e-9 * dmax)
        for i in np.flatnonzero(close):
            d = _norm3(gap[i])
            adm[i] = d > 0.0 and dmax[i] <= eta * d
        leaf_t = child[T, 0] < 0
        leaf_s = child[S, 0] < 0
        stop = adm | (leaf_t & leaf_s)
        out_t.append(T[stop]); out_s.append(S[stop]); out_adm.append(adm[stop])
        out_key.append(key[stop]); out_depth.append(np.full(int(stop.sum()), depth))
        T, S, key, lt, ls = T[~stop], S[~stop], key[~stop], leaf_t[~stop], leaf_s[~stop]
        nt, ns = [], []
        nkey = []
        for i in range(2):
            for j in range(2):
                m = (~lt if i == 1 else np.ones_like(lt)) & (~ls if j == 1 else np.ones_like(ls))
                tt = np.where(lt, T, child[T, i])[m]
                ss = np.where(ls, S, child[S, j])[m]
                nt.append(tt); ns.append(ss); nkey.append(key[m] * 4 + (2 * i + j))
        T, S, key = np.concatenate(nt), np.concatenate(ns), np.concatenate(nkey)
        depth += 1
    t = np.concatenate(out_t)
    s = np.concatenate(out_s)
    a = np.concatenate(out_adm)
    k = np.concatenate(out_key)
    d = np.concatenate(out_depth)
    maxd = int(d.max()) if d.size else 0
    if 2 * maxd > 62:
        raise ValueError("block tree too deep")
    order = np.argsort(k << (2 * (maxd - d)), kind="stable")
    return t[order], s[order], a[order]


# ---------------------------------------------------------------------------
# low-rank kernels (numpy, reference operation order)
# ---------------------------------------------------------------------------

def chebyshev_points(lo: np.ndarray, hi: np.ndarray, order: int) -> np.ndarray:
    if order < 1:
        raise ValueError("Chebyshev order must be >= 1")
    nodes = np.cos((2.0 * np.arange(order) + 1.0) * np.pi / (2.0 * order))
    axes = [0.5 * (lo[d] + hi[d]) + 0.5 * (hi[d] - lo[d]) * nodes for d in range(3)]
    return np.stack(np.meshgrid(*axes, indexing="ij"), axis=-1).reshape(-1, 3)


def green_cross(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    d = np.linalg.norm(np.atleast_2d(x)[:, None, :] - np.atleast_2d(y)[None, :, :], axis=2)
    if np.any(d == 0.0):
        raise ValueError("Green's function is singular at coincident points")
    return -1.0 / (_FOUR_PI * d)


def aca_full(s: np.ndarray, epsilon: float):
    """Fully pivoted cross of an explicit matrix (lowrank.py:125-150)."""
    res = np.array(s, dtype=np.float64, copy=True)
    norm0 = float(np.linalg.norm(res))
    tau: list[int] = []
    sigma: list[int] = []
    if norm0 != 0.0:
        cap = min(res.shape)
        floor = epsilon * norm0 / np.sqrt(res.size)
        while len(tau) < cap:
            i, j = divmod(int(np.argmax(np.abs(res))), res.shape[1])
            piv = res[i, j]
            if abs(piv) <= floor:
                break
            tau.append(i)
            sigma.append(j)
            res -= np.outer(res[:, j] / piv, res[i, :])
            if float(np.linalg.norm(res)) <= epsilon * norm0:
                break
    return np.array(tau, dtype=np.int64), np.array(sigma, dtype=np.int64)


def aca(row_eval, col_eval, n_rows: int, n_cols: int, epsilon: float, max_rank=None):
    """Partially pivoted ACA (lowrank.py:36-122); returns (a, b, converged)."""
    if epsilon <= 0.0:
        raise ValueError("epsilon must be positive")
    cap = min(n_rows, n_cols) if max_rank is None else min(max_rank, n_rows, n_cols)
    a_cols, b_cols = [], []
    used_rows: set[int] = set()
    frob_sq = 0.0
    next_row = 0
    converged = False
    while len(a_cols) < cap:
        pivot = None
        i = next_row
        for _ in range(n_rows):
            if i not in used_rows:
                orig = np.array(row_eval(i), dtype=np.float64)
                res_row = orig.copy()
                for a_l, b_l in zip(a_cols, b_cols):
                    res_row -= a_l[i] * b_l
                j = int(np.argmax(np.abs(res_row)))
                if abs(res_row[j]) > 1e-14 * (np.linalg.norm(orig) + np.sqrt(frob_sq)):
                    pivot = (i, j, res_row)
                    break
                used_rows.add(i)
            i = (i + 1) % n_rows
        if pivot is None:
            converged = True
            break
        i, j, res_row = pivot
        delta = res_row[j]
        res_col = np.array(col_eval(j), dtype=np.float64)
        for a_l, b_l in zip(a_cols, b_cols):
            res_col -= b_l[j] * a_l
        a_new = res_col / delta
        b_new = res_row
        na = float(np.linalg.norm(a_new))
        nb = float(np.linalg.norm(b_new))
        cross = 0.0
        for a_l, b_l in zip(a_cols, b_cols):
            cross += float(a_new @ a_l) * float(b_new @ b_l)
        frob_sq = max(frob_sq + na * na * nb * nb + 2.0 * cross, 0.0)
        a_cols.append(a_new)
        b_cols.append(b_new)
        used_rows.add(i)
        masked = np.abs(a_new).copy()
        masked[list(used_rows)] = -np.inf
        next_row = int(np.argmax(masked))
        if na * nb <= epsilon * np.sqrt(frob_sq):
            converged = True
            break
    k = len(a_cols)
    a = np.column_stack(a_cols) if k else np.zeros((n_rows, 0))
    b = np.column_stack(b_cols) if k else np.zeros((n_cols, 0))
    if k == cap and not converged and cap == min(n_rows, n_cols):
        converged = True
    return a, b, converged


def truncate_lowrank(a: np.ndarray, b: np.ndarray, epsilon: float):
    if a.shape[1] == 0:
        return a, b
    qa, ra = np.linalg.qr(a)
    qb, rb = np.linalg.qr(b)
    u, s, vt = np.linalg.svd(ra @ rb.T)
    if s.size == 0 or s[0] == 0.0:
        return a[:, :0], b[:, :0]
    keep = int(np.sum(s > epsilon * s[0]))
    return qa @ (u[:, :keep] * s[:keep]), qb @ vt[:keep].T


# ---------------------------------------------------------------------------
# collocation entries on the GPU
# ---------------------------------------------------------------------------

class GpuCollocation:
    """Entry evaluator backed by csrc/colloc.cu (h2b_colloc_* C ABI)."""

    def __init__(self, surface: Surface, panels: np.ndarray, inc):
        lib = nat.lib()
        for nm, args in (("h2b_colloc_create", [C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                                 C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]),
                         ("h2b_colloc_eval", [C.c_void_p, C.c_int64] + [C.c_void_p] * 5
                          + [C.c_int64, C.c_void_p, C.c_int64, C.c_void_p])):
            getattr(lib, nm).argtypes = args
            getattr(lib, nm).restype = C.c_int
        lib.h2b_colloc_destroy.argtypes = [C.c_void_p]
        lib.h2b_colloc_destroy.restype = None
        self._lib = lib
        inc_ptr, inc_tri, inc_loc = (np.ascontiguousarray(a) for a in inc)
        self._keep = (np.ascontiguousarray(panels, np.float64), inc_ptr, inc_tri,
                      np.ascontiguousarray(inc_loc, np.int8), np.ascontiguousarray(surface.diag))
        h = C.c_void_p()
        p, ip, it, il, dg = self._keep
        nat.check(lib.h2b_colloc_create(surface.n, p.shape[0], p.ctypes.data, ip.ctypes.data, it.ctypes.data,
                                        il.ctypes.data, dg.ctypes.data, C.byref(h)), "h2b_colloc_create")
        self._h = h

    def rows(self, points, col_begin, col_count, diag_node, out_off, colidx, out_len):
        pts = np.ascontiguousarray(points, np.float64)
        cb = np.ascontiguousarray(col_begin, np.int64)
        cc = np.ascontiguousarray(col_count, np.int32)
        dn = np.ascontiguousarray(diag_node, np.int64)
        oo = np.ascontiguousarray(out_off, np.int64)
        ci = np.ascontiguousarray(colidx, np.int64)
        out = np.empty(max(1, int(out_len)))
        nat.check(self._lib.h2b_colloc_eval(self._h, pts.shape[0], pts.ctypes.data, cb.ctypes.data,
                                            cc.ctypes.data, dn.ctypes.data, oo.ctypes.data, ci.size,
                                            ci.ctypes.data, int(out_len), out.ctypes.data), "h2b_colloc_eval")
        return out[:out_len]

    def close(self):
        if self._h:
            self._lib.h2b_colloc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# the build
# ---------------------------------------------------------------------------

@dataclass
class BuildReport:
    n: int = 0
    nclusters: int = 0
    n_admissible: int = 0
    n_dense: int = 0
    n_fallback: int = 0
    seconds: dict = None


_G: dict = {}  # state shared with the worker pool (sent once per worker)


def _worker_init(state: dict) -> None:
    _G.clear()
    _G.update(state)
    try:  # one BLAS thread per worker process
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass


def _pool(workers: int):
    # spawn, not fork: the parent usually holds a CUDA context and BLAS/driver
    # threads, and forking a multi-threaded process can deadlock the children
    import multiprocessing as mp
    import sys
    main = sys.modules.get("__main__")
    main_file = getattr(main, "__file__", None)
    hide = main_file is not None and not os.path.exists(main_file)   # e.g. `python -` (stdin)
    if hide:
        del main.__file__
    try:  # workers are started here; the main-module fixup happens now
        return mp.get_context("spawn").Pool(workers, initializer=_worker_init, initargs=(dict(_G),))
    finally:
        if hide:
            main.__file__ = main_file


def _hca_prepare(bi: int):
    """hca.py:38-105 up to (not including) the panel rows of B."""
    g = _G
    t, s = g["bt"][bi], g["bs"][bi]
    order, eps = g["order"], g["eps"]
    eta_t = chebyshev_points(g["lo"][t], g["hi"][t], order)
    eta_s = chebyshev_points(g["lo"][s], g["hi"][s], order)
    s_mat = green_cross(eta_t, eta_s)
    tau, sigma = aca_full(s_mat, eps)
    if tau.size == 0:
        return ("zero", None, None)
    cross = s_mat[np.ix_(tau, sigma)]
    if np.linalg.cond(cross) > _COND_LIMIT:
        return ("fallback", None, None)
    rows = g["perm"][g["start"][t]: g["end"][t]]
    g_cols = green_cross(g["coords"][rows], eta_s[sigma])
    a = np.linalg.solve(cross.T, g_cols.T).T
    return ("ok", a, eta_t[tau])


def _truncate(args):
    a, b = args
    return truncate_lowrank(a, b, _G["eps"])


def _map(fn, items, workers, chunksize=64):
    if workers <= 1 or len(items) < 2 * chunksize:
        return [fn(i) for i in items]
    with _pool(workers) as p:
        return p.map(fn, items, chunksize=chunksize)


def assemble_h2(surface: Surface, config: CompressionConfig = CompressionConfig(), *,
                evaluator=None, workers: int | None = None, log=None,
                backend: str = "numpy", device: str = "cuda",
                recompress_backend: str = "host") -> tuple[H2Matrix, BuildReport]:
    """Build the compressed operator M = K + D of ``surface`` as an H2Matrix
    (``hmatrix.assemble_operator(mesh, "h2", config).payload``).

    backend "numpy": the reference's operation order (bit-identical
    operators, tests/test_builder.py).  backend "gpu": the admissible blocks
    by batched HCA on the GPU (assembly/gpu_hca.py) and Gram-based bases in
    the recompression -- the same algorithm to rounding, for the large
    BASELINE workloads; with ``recompress_backend="gpu"`` the recompression
    itself runs on the device too (assembly/gpu_recompress.py, SURVEY §8f
    row 4)."""
    _say = log or (lambda *a: None)

    def say(msg):  # with the process's resident / peak memory
        try:
            import resource
            rss = int(open("/proc/self/statm").read().split()[1]) * os.sysconf("SC_PAGE_SIZE") / 1e9
            peak = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6
            _say(f"{msg} [rss {rss:.1f} GB, peak {peak:.1f} GB]")
        except (OSError, ValueError):
            _say(msg)
    times = {}
    t0 = time.perf_counter()
    workers = workers or max(1, min(32, os.cpu_count() or 1))
    panels = panel_table(surface)
    inc = incidence(surface)
    if evaluator is None:
        evaluator = GpuCollocation(surface, panels, inc)
    elif callable(evaluator):
        evaluator = evaluator(surface, panels, inc)
    coords = surface.coords
    tree = build_cluster_tree(coords, config.leaf_size)
    cl = tree.clusters
    start = np.array([c.start for c in cl], np.int64)
    end = np.array([c.end for c in cl], np.int64)
    lo = np.array([c.bbox_min for c in cl])
    hi = np.array([c.bbox_max for c in cl])
    perm = tree.perm
    bt, bs, badm = leaf_block_list(tree, config.eta)
    times["tree+blocks"] = time.perf_counter() - t0
    say(f"tree {len(cl)} clusters, {int(badm.sum())} admissible + {int((~badm).sum())} dense blocks "
        f"({times['tree+blocks']:.1f}s)")

    # ---- dense near field: one GPU row job per block row (bem.py:221-235)
    t1 = time.perf_counter()
    dense_ids = np.flatnonzero(~badm)
    dt, ds = bt[dense_ids], bs[dense_ids]
    rows_per = end[dt] - start[dt]
    cols_per = end[ds] - start[ds]
    sizes = rows_per * cols_per
    blk_off = np.zeros(dense_ids.size + 1, np.int64)
    np.cumsum(sizes, out=blk_off[1:])
    job_blk = np.repeat(np.arange(dense_ids.size), rows_per)
    job_row = np.arange(job_blk.size) - np.repeat(np.cumsum(rows_per) - rows_per, rows_per)
    row_node = perm[start[dt][job_blk] + job_row]
    near_flat = evaluator.rows(coords[row_node], start[ds][job_blk], cols_per[job_blk].astype(np.int32),
                               row_node, blk_off[job_blk] + job_row * cols_per[job_blk], perm,
                               int(blk_off[-1]))
    near_mats = [near_flat[blk_off[i]: blk_off[i + 1]].reshape(rows_per[i], cols_per[i])
                 for i in range(dense_ids.size)]
    times["near"] = time.perf_counter() - t1
    say(f"near field: {dense_ids.size} blocks, {blk_off[-1] * 8 / 1e6:.1f} MB ({times['near']:.1f}s)")

    # ---- admissible blocks: HCA (hca.py:38-105)
    t2 = time.perf_counter()
    adm_ids = np.flatnonzero(badm)
    _G.clear()
    _G.update(bt=bt[adm_ids], bs=bs[adm_ids], lo=lo, hi=hi, start=start, end=end, perm=perm,
              coords=coords, order=config.cheb_order, eps=config.eps)
    weights = None
    if backend == "gpu" and config.method == "hca":
        from .gpu_hca import FactorArena, hca_gpu
        lowrank, weights, n_fb = [None] * adm_ids.size, [None] * adm_ids.size, 0
        arena = FactorArena()
        # in chunks of blocks: the raw (untruncated) factors of one chunk at a
        # time, the truncated ones packed into the arena (host-memory bound of
        # the 4M-node build)
        chunk = int(os.environ.get("H2B_HCA_CHUNK", "65536"))
        for c0 in range(0, adm_ids.size, chunk):
            ids = adm_ids[c0:c0 + chunk]
            res = hca_gpu(bt=bt[ids], bs=bs[ids], lo=lo, hi=hi, start=start, end=end, perm=perm,
                          coords=coords, order=config.cheb_order, eps=config.eps, evaluator=evaluator,
                          device=device, times=times, arena=arena)
            for j, (st, a, b) in enumerate(res):
                i = c0 + j
                t_c, s_c = int(bt[adm_ids[i]]), int(bs[adm_ids[i]])
                if st == "ok":
                    lowrank[i] = (a, b)
                    # a = Q_a U S, b = Q_b V: B^T B = I, A^T A = S^2 (see recompress):
                    # identity and diagonal weights
                    weights[i] = (None, np.linalg.norm(a, axis=0))
                    continue
                if st == "zero":
                    lowrank[i] = (np.zeros((end[t_c] - start[t_c], 0)), np.zeros((end[s_c] - start[s_c], 0)))
                else:
                    warnings.warn("ill-conditioned interpolation cross; falling back to ACA", RuntimeWarning)
                    n_fb += 1
                    lowrank[i] = _aca_block(evaluator, coords, perm, start, end, t_c, s_c, config.eps)
                aa, bb = lowrank[i]
                weights[i] = (np.linalg.qr(bb)[1], np.linalg.qr(aa)[1])
            del res
            if c0 == 0 or (c0 // chunk) % 8 == 7:
                say(f"HCA (gpu): {min(adm_ids.size, c0 + chunk)} / {adm_ids.size} blocks")
        times["hca_gpu"] = time.perf_counter() - t2
        fbytes = sum(a.nbytes + b.nbytes for a, b in lowrank)
        times["factor_gb"] = fbytes / 1e9
        say(f"HCA (gpu): {adm_ids.size} blocks, factors {fbytes / 1e9:.2f} GB, {n_fb} ACA fallbacks ({times['hca_gpu']:.1f}s: "
            + ", ".join(f"{k} {times[k]:.1f}s" for k in ("cross", "solve", "rows", "truncate") if k in times) + ")")
        t5 = time.perf_counter()
        lr_list = [(int(bt[adm_ids[i]]), int(bs[adm_ids[i]]), lowrank[i][0], lowrank[i][1])
                   for i in range(adm_ids.size)]
        dense_list = [(int(dt[i]), int(ds[i]), near_mats[i]) for i in range(dense_ids.size)]
        if recompress_backend == "gpu":
            from .gpu_recompress import recompress_gpu
            op = recompress_gpu(tree, surface.n, lr_list, dense_list, config.eps_rec, weights, timings=times)
            times["recompress"] = time.perf_counter() - t5
            times["total"] = time.perf_counter() - t0
            say(f"recompress (gpu) {times['recompress']:.1f}s (rows: pack {times.get('rec_rows_pack', 0):.1f}s, levels "
                f"{times.get('rec_rows', 0):.1f}s; cols: pack {times.get('rec_cols_pack', 0):.1f}s, levels "
                f"{times.get('rec_cols', 0):.1f}s; coupling {times.get('rec_coupling', 0):.1f}s); "
                f"H² {op.storage_bytes() / 1e6:.1f} MB; total {times['total']:.1f}s")
        elif recompress_backend == "host":
            from .recompress import recompress
            op = recompress(tree, surface.n, lr_list, dense_list, config.eps_rec, workers=workers, weights=weights,
                            timings=times)
            times["recompress"] = time.perf_counter() - t5
            times["total"] = time.perf_counter() - t0
            say(f"recompress {times['recompress']:.1f}s (bases rows {times.get('rec_rows', 0):.1f}s, cols "
                f"{times.get('rec_cols', 0):.1f}s [weighting {times.get('rec_cols_weighting', 0):.1f}s, leaves "
                f"{times.get('rec_cols_leaf_cpu', 0):.1f} / inner {times.get('rec_cols_inner_cpu', 0):.1f} thread-s], coupling "
                f"{times.get('rec_coupling', 0):.1f}s); "
                f"H² {op.storage_bytes() / 1e6:.1f} MB; total {times['total']:.1f}s")
        else:
            raise ValueError(f"unknown recompress_backend {recompress_backend!r}")
        rep = BuildReport(n=surface.n, nclusters=len(cl), n_admissible=int(adm_ids.size),
                          n_dense=int(dense_ids.size), n_fallback=n_fb, seconds=times)
        return op, rep
    if config.method == "hca":
        prep = _map(_hca_prepare, list(range(adm_ids.size)), workers)
    else:
        prep = [("fallback", None, None)] * adm_ids.size
    times["hca_cross"] = time.perf_counter() - t2
    # B = panel rows at the interpolation pivots (bem.py:207-219), one GPU batch
    t3 = time.perf_counter()
    ok = [i for i, p in enumerate(prep) if p[0] == "ok"]
    kk = np.array([prep[i][2].shape[0] for i in ok], np.int64)
    ss = adm_ids[ok] if ok else np.zeros(0, np.int64)
    s_cl = bs[ss]
    ncol = (end[s_cl] - start[s_cl])
    job_cnt = np.repeat(ncol, kk)
    pts = np.concatenate([prep[i][2] for i in ok]) if ok else np.zeros((0, 3))
    job_cb = np.repeat(start[s_cl], kk)
    job_off = np.zeros(job_cnt.size + 1, np.int64)
    np.cumsum(job_cnt, out=job_off[1:])
    bflat = evaluator.rows(pts, job_cb, job_cnt.astype(np.int32), np.full(job_cnt.size, -1, np.int64),
                           job_off[:-1], perm, int(job_off[-1]))
    lowrank = [None] * adm_ids.size
    pend = []
    jo = 0
    for q, i in enumerate(ok):
        k, m = int(kk[q]), int(ncol[q])
        b = bflat[job_off[jo]: job_off[jo] + k * m].reshape(k, m).T
        jo += k
        pend.append((i, prep[i][1], b))
    times["hca_rows"] = time.perf_counter() - t3
    t4 = time.perf_counter()
    trunc = _map(_truncate, [(a, b) for _, a, b in pend], workers, chunksize=256)
    for (i, _, _), ab in zip(pend, trunc):
        lowrank[i] = ab
    n_fb = 0
    for i, p in enumerate(prep):
        t_c, s_c = int(bt[adm_ids[i]]), int(bs[adm_ids[i]])
        if p[0] == "zero":
            lowrank[i] = (np.zeros((end[t_c] - start[t_c], 0)), np.zeros((end[s_c] - start[s_c], 0)))
        elif p[0] == "fallback":
            if config.method == "hca":
                warnings.warn("ill-conditioned interpolation cross; falling back to ACA", RuntimeWarning)
            n_fb += 1
            lowrank[i] = _aca_block(evaluator, coords, perm, start, end, t_c, s_c, config.eps)
    times["hca_trunc"] = time.perf_counter() - t4
    say(f"HCA: {adm_ids.size} blocks, {n_fb} ACA fallbacks "
        f"(cross {times['hca_cross']:.1f}s, rows {times['hca_rows']:.1f}s, trunc {times['hca_trunc']:.1f}s)")

    # ---- H -> H² (h2.py:148-183)
    t5 = time.perf_counter()
    from .recompress import recompress
    op = recompress(tree, surface.n, [(int(bt[adm_ids[i]]), int(bs[adm_ids[i]]), lowrank[i][0], lowrank[i][1])
                                      for i in range(adm_ids.size)],
                    [(int(dt[i]), int(ds[i]), near_mats[i]) for i in range(dense_ids.size)],
                    config.eps_rec, workers=workers)
    times["recompress"] = time.perf_counter() - t5
    times["total"] = time.perf_counter() - t0
    say(f"recompress {times['recompress']:.1f}s; H² {op.storage_bytes() / 1e6:.1f} MB; total {times['total']:.1f}s")
    rep = BuildReport(n=surface.n, nclusters=len(cl), n_admissible=int(adm_ids.size),
                      n_dense=int(dense_ids.size), n_fallback=n_fb, seconds=times)
    return op, rep


def _aca_block(evaluator, coords, perm, start, end, t, s, eps):
    """aca_block (hca.py:19-35): partially pivoted ACA on the block itself."""
    rows = perm[start[t]:end[t]]
    cols = perm[start[s]:end[s]]

    def row_eval(i):
        return evaluator.rows(coords[rows[i]][None, :], np.array([start[s]]), np.array([cols.size], np.int32),
                              np.array([-1]), np.array([0]), perm, cols.size)

    def col_eval(j):
        nr = rows.size
        return evaluator.rows(coords[rows], np.full(nr, start[s] + j), np.ones(nr, np.int32),
                              rows, np.arange(nr), perm, nr)

    a, b, conv = aca(row_eval, col_eval, rows.size, cols.size, eps)
    return a, b
