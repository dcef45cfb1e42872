"""H² operator data model and the drop-in GPU ``h2_matvec``.

Reference interface being replaced (all /root/reference/pkg/src/strayfield):

* ``h2_matvec(op, x)``            hmatrix/h2.py:186-244
* ``H2Matrix.matvec(self, x)``    hmatrix/h2.py:74-75 (module-global lookup)
* ``H2Matrix.storage_bytes()``    hmatrix/h2.py:77-83
* ``H2Matrix.row_rank/col_rank``  hmatrix/h2.py:44-54

``h2_matvec`` keeps the reference's signature and contract: ``x`` is coerced
with ``np.asarray(x, dtype=float64)``; any shape other than ``(op.n,)`` raises
``ValueError("vector must have shape (n,)")``; a fresh array in original node
order is returned; ``x`` and ``op`` are never mutated.  The product runs in
libh2b.so (one persistent sm_100a kernel); there is no CPU
fallback.  The device copy of an operator is cached per operator object
(``H2Matrix`` is ``eq=False``, hence identity-hashable), its options and a
structural fingerprint (replaced or resized block lists/dicts rebuild it);
a matrix edited in place after the first product needs ``invalidate(op)``
-- the reference treats operators as immutable.
"""

from __future__ import annotations

import ctypes as C
import threading
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .cluster import ClusterTree

__all__ = ["H2Matrix", "h2_matvec", "h2_matmat", "DeviceOperator", "device_operator", "invalidate",
           "describe", "plan_view", "install_into_reference", "rank_arrays", "nccl_unique_id"]


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 creates it, every rank passes it to
    ``DeviceOperator(op, rank=r, world_size=W, nccl_unique_id=...)``)."""
    buf = C.create_string_buffer(128)
    nat.check(nat.lib().h2b_nccl_unique_id(buf), "h2b_nccl_unique_id")
    return buf.raw


@dataclass(eq=False)
class H2Matrix:
    """Nested-basis operator with the reference's field layout
    (hmatrix/h2.py:23-42): per-cluster dicts keyed by preorder id, coupling
    and near-field block lists ``(row_cid, col_cid, matrix)``."""

    tree: ClusterTree
    n: int
    row_basis: dict[int, np.ndarray] = field(default_factory=dict)
    row_transfer: dict[int, np.ndarray] = field(default_factory=dict)
    col_basis: dict[int, np.ndarray] = field(default_factory=dict)
    col_transfer: dict[int, np.ndarray] = field(default_factory=dict)
    coupling: list[tuple[int, int, np.ndarray]] = field(default_factory=list)
    near: list[tuple[int, int, np.ndarray]] = field(default_factory=list)

    def row_rank(self, cid: int) -> int:
        c = self.tree.clusters[cid]
        if c.is_leaf:
            return self.row_basis[cid].shape[1]
        return self.row_transfer[c.children[0].cid].shape[1]

    def col_rank(self, cid: int) -> int:
        c = self.tree.clusters[cid]
        if c.is_leaf:
            return self.col_basis[cid].shape[1]
        return self.col_transfer[c.children[0].cid].shape[1]

    def explicit_row_basis(self, cid: int) -> np.ndarray:
        c = self.tree.clusters[cid]
        if c.is_leaf:
            return self.row_basis[cid]
        return np.vstack([self.explicit_row_basis(ch.cid) @ self.row_transfer[ch.cid]
                          for ch in c.children])

    def explicit_col_basis(self, cid: int) -> np.ndarray:
        c = self.tree.clusters[cid]
        if c.is_leaf:
            return self.col_basis[cid]
        return np.vstack([self.explicit_col_basis(ch.cid) @ self.col_transfer[ch.cid]
                          for ch in c.children])

    def matvec(self, x: np.ndarray) -> np.ndarray:
        return h2_matvec(self, x)

    def storage_bytes(self) -> int:
        total = 0
        for d in (self.row_basis, self.row_transfer, self.col_basis, self.col_transfer):
            total += sum(m.size for m in d.values())
        total += sum(s.size for _, _, s in self.coupling)
        total += sum(m.size for _, _, m in self.near)
        return total * 8


def rank_arrays(op) -> tuple[np.ndarray, np.ndarray]:
    """Per-cluster (k_row, k_col), the reference's row_rank/col_rank
    (h2.py:44-54) for every preorder id."""
    nc = len(op.tree.clusters)
    k_row = np.zeros(nc, np.int64)
    k_col = np.zeros(nc, np.int64)
    for c in op.tree.clusters:
        if c.is_leaf:
            k_row[c.cid] = op.row_basis[c.cid].shape[1]
            k_col[c.cid] = op.col_basis[c.cid].shape[1]
        else:
            k_row[c.cid] = op.row_transfer[c.children[0].cid].shape[1]
            k_col[c.cid] = op.col_transfer[c.children[0].cid].shape[1]
    return k_row, k_col


class _DescHolder:
    """A filled ``h2b_desc`` plus the numpy arrays its pointers refer to."""

    def __init__(self, op):
        from .cluster import tree_arrays
        ta = tree_arrays(op.tree)
        n = int(op.n)
        if ta["perm"].shape != (n,):
            raise ValueError("tree.perm does not match op.n")
        nc = ta["cl_start"].shape[0]
        k_row, k_col = rank_arrays(op)
        keep = []

        def cont(m):
            a = np.ascontiguousarray(m, dtype=np.float64)
            keep.append(a)
            return a

        rb = [None] * nc
        cb = [None] * nc
        rt = [None] * nc
        ct = [None] * nc
        for cid, m in op.row_basis.items():
            rb[cid] = cont(m)
        for cid, m in op.col_basis.items():
            cb[cid] = cont(m)
        for cid, m in op.row_transfer.items():
            rt[cid] = cont(m)
        for cid, m in op.col_transfer.items():
            ct[cid] = cont(m)
        cp_row = np.array([b[0] for b in op.coupling], np.int64)
        cp_col = np.array([b[1] for b in op.coupling], np.int64)
        cp = [cont(b[2]) for b in op.coupling]
        nr_row = np.array([b[0] for b in op.near], np.int64)
        nr_col = np.array([b[1] for b in op.near], np.int64)
        nr = [cont(b[2]) for b in op.near]
        # shape checks against the tree (cheap, catches malformed payloads)
        size = ta["cl_end"] - ta["cl_start"]
        for (r, s), m in zip(zip(nr_row, nr_col), nr):
            if m.shape != (size[r], size[s]):
                raise ValueError(f"near block ({r},{s}) has shape {m.shape}, expected {(size[r], size[s])}")
        for (r, s), m in zip(zip(cp_row, cp_col), cp):
            if m.shape != (k_row[r], k_col[s]):
                raise ValueError(f"coupling block ({r},{s}) has shape {m.shape}")
        self.arrays = dict(ta, k_row=k_row, k_col=k_col, cp_row=cp_row, cp_col=cp_col,
                           nr_row=nr_row, nr_col=nr_col)
        self.keep = keep
        self.ptrs = [nat.ptr_array(rb), nat.ptr_array(cb), nat.ptr_array(rt), nat.ptr_array(ct),
                     nat.ptr_array(cp), nat.ptr_array(nr)]
        a = self.arrays
        d = nat.Desc()
        d.n = n
        d.nclusters = nc
        d.perm = nat.as_i64_ptr(a["perm"])
        d.cl_start = nat.as_i64_ptr(a["cl_start"])
        d.cl_end = nat.as_i64_ptr(a["cl_end"])
        d.cl_child = nat.as_i64_ptr(np.ascontiguousarray(a["cl_child"]))
        d.k_row = nat.as_i64_ptr(k_row)
        d.k_col = nat.as_i64_ptr(k_col)
        d.row_basis, d.col_basis, d.row_transfer, d.col_transfer = self.ptrs[:4]
        d.ncoupling = len(op.coupling)
        d.cp_row = nat.as_i64_ptr(cp_row)
        d.cp_col = nat.as_i64_ptr(cp_col)
        d.cp_data = self.ptrs[4]
        d.nnear = len(op.near)
        d.nr_row = nat.as_i64_ptr(nr_row)
        d.nr_col = nat.as_i64_ptr(nr_col)
        d.nr_data = self.ptrs[5]
        self.desc = d


def describe(op) -> _DescHolder:
    """Flatten a (reference or mirror) H2Matrix into an ``h2b_desc``."""
    return _DescHolder(op)


# h2b_options.sched_flags bits (include/h2b.h)
SCHED_NEAR_FIRST = 1
SCHED_EXPLICIT = 8
SCHED_NO_RING = 1 << 24


def SCHED_LEAF_MIX(m: int) -> int:
    return (int(m) & 0xF) << 20


def SCHED_RING_WARPS(k: int) -> int:
    return (int(k) & 0xF) << 4


def SCHED_NEAR_PRIO(k: int) -> int:
    return (int(k) & 0xF) << 26


PLAN_SKIP_LEVELS = 1
PLAN_NO_SKIP = 2
PLAN_NEAR_SPLIT = 4
PLAN_GATE = 1 << 8
PLAN_NO_GATE = 1 << 9
PLAN_STAGED = 1 << 10
PLAN_NO_STAGED = 1 << 11


def PLAN_SWEEP_NODES(v: int) -> int:
    """Bottom subtrees of at most 64 << v nodes (plan_flags bits 12-15)."""
    return (int(v) & 0xF) << 12


def _options(task_bytes=0, far_task_bytes=0, warps_per_cta=0, ctas_per_sm=0, max_nrhs=0, sched_flags=0,
             band_depth=0, rank=0, world_size=1, nccl_unique_id=None, near_phase0_pct=0,
             plan_flags=0) -> nat.Options:
    o = nat.Options()
    o.task_bytes = int(task_bytes)
    o.far_task_bytes = int(far_task_bytes)
    o.warps_per_cta = int(warps_per_cta)
    o.ctas_per_sm = int(ctas_per_sm)
    o.max_nrhs = int(max_nrhs)
    o.sched_flags = int(sched_flags)
    o.band_depth = int(band_depth)
    o.rank = int(rank)
    o.world_size = int(world_size)
    o.near_phase0_pct = int(near_phase0_pct)
    o.plan_flags = int(plan_flags)
    if nccl_unique_id is not None:
        buf = C.create_string_buffer(bytes(nccl_unique_id), 128)
        o._keep_id = buf
        o.nccl_unique_id = C.cast(buf, C.c_void_p)
    return o


def _grab_view(v) -> dict:
    T, S, D = v.ntasks, v.nsegs, v.ndeps

    def grab(ptr, count, dtype):
        if count == 0:
            return np.zeros(0, dtype)
        return np.ctypeslib.as_array(ptr, shape=(count,)).astype(dtype, copy=True)

    return {
        "coef_len": int(v.coef_len),
        "t_data": grab(v.t_data, T, np.int64), "t_out": grab(v.t_out, T, np.int64),
        "t_bias": grab(v.t_bias, T, np.int64), "t_m": grab(v.t_m, T, np.int32),
        "t_ld": grab(v.t_ld, T, np.int32), "t_ncols": grab(v.t_ncols, T, np.int32),
        "t_kind": grab(v.t_kind, T, np.int32), "t_seg0": grab(v.t_seg0, T + 1, np.int32),
        "t_dep0": grab(v.t_dep0, T + 1, np.int32),
        "t_bias_nslots": grab(v.t_bias_nslots, T, np.int32),
        "t_bias_stride": grab(v.t_bias_stride, T, np.int32),
        "s_src": grab(v.s_src, S, np.int64), "s_ncols": grab(v.s_ncols, S, np.int32),
        "s_kind": grab(v.s_kind, S, np.int32), "s_nslots": grab(v.s_nslots, S, np.int32),
        "s_stride": grab(v.s_stride, S, np.int32), "deps": grab(v.deps, D, np.int32),
        "t_mlen": grab(v.t_mlen, T, np.int32),
        "gated": grab(v.gated, int(v.ngated), np.int32), "n_gated1": int(v.n_gated1), "n_up": int(v.n_up),
        "mode": int(v.mode), "group": int(v.group), "split": int(v.split),
        "unit0": grab(v.unit0, int(v.nunits) + 1, np.int32) if v.mode == 1 else np.zeros(0, np.int32),
        "wave0": grab(v.wave0, int(v.nwaves) + 1, np.int32) if v.mode == 1 else np.zeros(0, np.int32),
        "resident": bool(v.resident),
        "res_max": (int(v.res_mat_max), int(v.res_vec_max), int(v.res_items_max)),
        "u_range": (grab(v.u_range, 8 * int(v.nunits), np.int64).reshape(-1, 8) if v.mode == 1
                    else np.zeros((0, 8), np.int64)),
    }


def plan_view(op, **options) -> dict:
    """Host-only execution plan (no GPU needed), returned as numpy copies:
    the arrays the kernel consumes plus stats.  Used by the CPU tests, which
    execute the plan with a numpy interpreter (oracle/flat_matvec.py).
    The top-level arrays are phase 0; ``phases`` lists every phase (two for
    a multi-GPU rank plan)."""
    h = describe(op)
    lib = nat.lib()
    handle = C.c_void_p()
    nat.check(lib.h2b_plan_create(C.byref(h.desc), C.byref(_options(**options)), C.byref(handle)),
              "h2b_plan_create")
    try:
        st = nat.Stats()
        nat.check(lib.h2b_plan_stats(handle, C.byref(st)))
        phases = []
        mat = None
        for k in range(lib.h2b_plan_phases(handle)):
            v = nat.PlanView()
            nat.check(lib.h2b_plan_phase_view(handle, k, C.byref(v)))
            if mat is None:
                mat = (np.ctypeslib.as_array(v.mat, shape=(v.mat_len,)).copy() if v.mat_len
                       else np.zeros(0))
            phases.append(_grab_view(v))
        world = max(1, int(options.get("world_size", 1)))
        lohi = np.zeros(2 * world, np.int64)
        exch = np.zeros(2, np.int64)
        nat.check(lib.h2b_plan_partition(handle, nat.as_i64_ptr(lohi), nat.as_i64_ptr(exch)))
        perm = np.ascontiguousarray(h.arrays["perm"]).copy()
        for ph in phases:
            ph.update(mat=mat, perm=perm, n=int(op.n))
        out = dict(phases[0])
        out.update(phases=phases, stats=st.as_dict(), rank_lo_hi=lohi.reshape(world, 2),
                   exchange=(int(exch[0]), int(exch[1])))
        return out
    finally:
        lib.h2b_plan_destroy(handle)


def _pinned_empty(shape) -> np.ndarray:
    """A fresh float64 host array in page-locked memory, so the product's
    device-to-host copy is one DMA.  The memory comes from torch's caching
    host allocator (no cudaHostAlloc per call) and returns to it when the
    array is released."""
    import torch
    return torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()


class DeviceOperator:
    """An H² operator resident on the current CUDA device (``h2b_op``)."""

    def __init__(self, op, **options):
        h = describe(op)
        self._create(h.desc, options)

    def _create(self, desc, options) -> None:
        self.n = int(desc.n)
        self._lib = nat.lib()
        handle = C.c_void_p()
        opts = _options(**options)
        nat.check(self._lib.h2b_create(C.byref(desc), C.byref(opts), C.byref(handle)), "h2b_create")
        self._h = handle
        self._lock = threading.Lock()

    @classmethod
    def from_desc(cls, desc, **options) -> "DeviceOperator":
        """From a filled ``h2b_desc`` (e.g. an opened H2MS file's)."""
        self = cls.__new__(cls)
        self._create(desc, options)
        return self

    def stats(self) -> dict:
        st = nat.Stats()
        nat.check(self._lib.h2b_stats_get(self._h, C.byref(st)))
        return st.as_dict()

    def stream_bytes(self) -> int:
        return int(self._lib.h2b_stream_bytes(self._h))

    def matvec(self, x: np.ndarray) -> np.ndarray:
        """Host arrays in/out: (n,) or (n, nrhs) with nrhs in {1,2,4,8,16}."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        nrhs = 1 if x.ndim == 1 else x.shape[1]
        y = _pinned_empty(x.shape)
        with self._lock:
            nat.check(self._lib.h2b_matvec(self._h, nat.as_d_ptr(x), nat.as_d_ptr(y),
                                           self.n, nrhs), "h2b_matvec")
        return y

    def matvec_dev(self, x_ptr: int, y_ptr: int, nrhs: int = 1, stream: int = 0) -> None:
        """Device pointers (e.g. ``tensor.data_ptr()``); asynchronous on ``stream``.
        For a multi-GPU rank operator, y receives this rank's rows."""
        nat.check(self._lib.h2b_matvec_dev(self._h, C.c_void_p(x_ptr), C.c_void_p(y_ptr),
                                           int(nrhs), C.c_void_p(stream)), "h2b_matvec_dev")

    LAUNCH_KINDS = {-1: "h2b_permute_kernel", 0: "h2b_dataflow_kernel", 1: "h2b_sweep_kernel", 2: "h2b_near_tma_kernel"}

    def launches(self, nrhs: int = 1) -> list:
        """The kernel launches of one product: kind, work items, matrix bytes."""
        out = []
        for k in range(self._lib.h2b_launch_count(self._h, int(nrhs))):
            kind, items, nbytes = np.zeros(1, np.int32), np.zeros(1, np.int64), np.zeros(1, np.int64)
            nat.check(self._lib.h2b_launch_info(self._h, int(nrhs), k, kind.ctypes.data_as(nat._p32),
                                                nat.as_i64_ptr(items), nat.as_i64_ptr(nbytes)))
            out.append({"kernel": self.LAUNCH_KINDS[int(kind[0])], "items": int(items[0]), "bytes": int(nbytes[0])})
        return out

    def launch_times(self, x_ptr: int, y_ptr: int, nrhs: int = 1, steps: int = 10, stream: int = 0) -> list:
        """Mean device milliseconds of every launch of a product (CUDA events
        around each launch; measurement aid, single GPU)."""
        info = self.launches(nrhs)
        ms = np.zeros(len(info))
        nat.check(self._lib.h2b_launch_times(self._h, C.c_void_p(x_ptr), C.c_void_p(y_ptr), int(nrhs), int(steps),
                                             C.c_void_p(stream), nat.as_d_ptr(ms)), "h2b_launch_times")
        for d, t in zip(info, ms):
            d["ms"] = float(t)
        return info

    def reset(self) -> None:
        """Scheduler state back to the just-created one (``h2b_reset``)."""
        nat.check(self._lib.h2b_reset(self._h), "h2b_reset")

    def matvec_phase(self, phase: int, x_ptr: int, y_ptr: int, nrhs: int = 1, stream: int = 0) -> None:
        """One phase of a multi-GPU rank product."""
        nat.check(self._lib.h2b_matvec_phase(self._h, int(phase), C.c_void_p(x_ptr), C.c_void_p(y_ptr),
                                             int(nrhs), C.c_void_p(stream)), "h2b_matvec_phase")

    def exchange_copy_from(self, other: "DeviceOperator", nrhs: int = 1, stream: int = 0) -> None:
        """Copy ``other``'s own x^ exchange region into this operator (for
        drivers that run the ranks' phases themselves)."""
        nat.check(self._lib.h2b_exchange_copy(self._h, other._h, int(nrhs), C.c_void_p(stream)),
                  "h2b_exchange_copy")

    def exchange_region(self, nrhs: int = 1) -> tuple[int, int]:
        """(device address, doubles per rank) of the x^ exchange regions."""
        base = C.c_void_p()
        cnt = np.zeros(1, np.int64)
        nat.check(self._lib.h2b_exchange_region(self._h, int(nrhs), C.byref(base), nat.as_i64_ptr(cnt)))
        return int(base.value or 0), int(cnt[0])

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.h2b_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_cache: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()
_cache_lock = threading.Lock()


def _fingerprint(op, options) -> tuple:
    """Cheap structural key of an operator's payload: which containers it
    holds and how many entries (catches replaced or resized lists/dicts;
    in-place edits of a matrix are not detected -- call ``invalidate``)."""
    parts = [int(op.n), id(op.tree)]
    for d in (op.row_basis, op.row_transfer, op.col_basis, op.col_transfer, op.coupling, op.near):
        parts += [id(d), len(d)]
    return tuple(parts) + tuple(sorted(options.items()))


def device_operator(op, **options) -> DeviceOperator:
    """Cached device copy of ``op`` (created on first use, keyed by the
    operator object, the options and a structural fingerprint).  The
    reference treats operators as immutable; after editing a
    matrix in place call ``invalidate(op)``."""
    key = _fingerprint(op, options)
    with _cache_lock:
        hit = _cache.get(op)
        if hit is not None and hit[0] == key:
            return hit[1]
        if hit is not None:
            hit[1].close()
        dev = DeviceOperator(op, **options)
        _cache[op] = (key, dev)
        return dev


def invalidate(op) -> None:
    """Drop the cached device copy of ``op`` (the next product re-uploads)."""
    with _cache_lock:
        hit = _cache.pop(op, None)
    if hit is not None:
        hit[1].close()


def h2_matvec(op, x: np.ndarray) -> np.ndarray:
    """Drop-in for the reference ``h2_matvec`` (h2.py:186-244), on the GPU."""
    x = np.asarray(x, dtype=np.float64)
    if x.shape != (op.n,):
        raise ValueError(f"vector must have shape ({op.n},)")
    return device_operator(op).matvec(x)


def h2_matmat(op, X: np.ndarray) -> np.ndarray:
    """Multi-RHS product Y = M X, X of shape (n, nrhs), nrhs in {1,2,4,8,16}.
    The reference has no such entry point (it rejects 2-D input); this is the
    batched form of ``h2_matvec`` applied column by column."""
    X = np.asarray(X, dtype=np.float64)
    if X.ndim != 2 or X.shape[0] != op.n:
        raise ValueError(f"matrix must have shape ({op.n}, nrhs)")
    return device_operator(op).matvec(X)


def install_into_reference(h2_module, package_module=None) -> None:
    """Route the reference's ``H2Matrix.matvec`` (which looks up the
    module-global ``h2_matvec`` at call time, h2.py:74-75) to the GPU path.
    Patch both ``strayfield.hmatrix.h2`` and the re-export in
    ``strayfield.hmatrix`` (hmatrix/__init__.py:13)."""
    h2_module.h2_matvec = h2_matvec
    if package_module is not None:
        package_module.h2_matvec = h2_matvec
