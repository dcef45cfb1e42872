"""ctypes binding of libh2b.so (the C ABI declared in include/h2b.h).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc,
sm_100a).  There is no fallback: if the shared object is missing, importing
any GPU entry point raises ``RuntimeError``.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

__all__ = ["lib", "Desc", "Options", "Stats", "PlanView", "check", "LIB_PATH",
           "KIND_NAMES", "H2BError"]

# H2B_LIB: an alternative build of the library (A/B timing of kernel variants)
LIB_PATH = Path(os.environ.get("H2B_LIB") or Path(__file__).resolve().parent / "libh2b.so")

ABI_VERSION = 4  # include/h2b.h H2B_ABI_VERSION
H2B_OK, H2B_EINVAL, H2B_ECUDA, H2B_ENCCL, H2B_ENOMEM, H2B_ENODEV, H2B_EIO, H2B_ECONV = 0, -1, -2, -3, -4, -5, -6, -7
KIND_NAMES = ("up_leaf", "up_node", "down", "near", "final")

_p64 = C.POINTER(C.c_int64)
_p32 = C.POINTER(C.c_int32)
_pd = C.POINTER(C.c_double)
_ppd = C.POINTER(_pd)


class Desc(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("nclusters", C.c_int64),
        ("perm", _p64), ("cl_start", _p64), ("cl_end", _p64), ("cl_child", _p64),
        ("k_row", _p64), ("k_col", _p64),
        ("row_basis", _ppd), ("col_basis", _ppd), ("row_transfer", _ppd), ("col_transfer", _ppd),
        ("ncoupling", C.c_int64), ("cp_row", _p64), ("cp_col", _p64), ("cp_data", _ppd),
        ("nnear", C.c_int64), ("nr_row", _p64), ("nr_col", _p64), ("nr_data", _ppd),
    ]


class Options(C.Structure):
    _fields_ = [
        ("task_bytes", C.c_int64), ("far_task_bytes", C.c_int64), ("warps_per_cta", C.c_int32), ("ctas_per_sm", C.c_int32),
        ("max_nrhs", C.c_int32), ("sched_flags", C.c_int32), ("band_depth", C.c_int32),
        ("rank", C.c_int32), ("world_size", C.c_int32), ("nccl_unique_id", C.c_void_p),
        ("near_phase0_pct", C.c_int32), ("plan_flags", C.c_int32),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("stream_bytes", C.c_int64), ("pool_bytes", C.c_int64),
        ("coef_doubles", C.c_int64), ("ntasks", C.c_int64), ("nsegs", C.c_int64),
        ("ndeps", C.c_int64), ("tasks_by_kind", C.c_int64 * 5), ("bytes_by_kind", C.c_int64 * 5),
        ("grid", C.c_int32), ("warps_per_cta", C.c_int32), ("rank", C.c_int32),
        ("world_size", C.c_int32), ("local_bytes", C.c_int64),
        ("sched_flags", C.c_int32), ("ring_warps", C.c_int32), ("extra_bytes", C.c_int64),
        ("launches", C.c_int32), ("resident_mask", C.c_int32),
    ]

    def as_dict(self) -> dict:
        d = {f: getattr(self, f) for f, _ in self._fields_
             if f not in ("tasks_by_kind", "bytes_by_kind")}
        d["tasks_by_kind"] = dict(zip(KIND_NAMES, list(self.tasks_by_kind)))
        d["bytes_by_kind"] = dict(zip(KIND_NAMES, list(self.bytes_by_kind)))
        return d


class PlanView(C.Structure):
    _fields_ = [
        ("ntasks", C.c_int64), ("nsegs", C.c_int64), ("ndeps", C.c_int64),
        ("mat_len", C.c_int64), ("coef_len", C.c_int64),
        ("mat", _pd), ("t_data", _p64), ("t_out", _p64), ("t_bias", _p64),
        ("t_m", _p32), ("t_ld", _p32), ("t_ncols", _p32), ("t_kind", _p32),
        ("t_seg0", _p32), ("t_dep0", _p32), ("t_bias_nslots", _p32), ("t_bias_stride", _p32),
        ("s_src", _p64), ("s_ncols", _p32), ("s_kind", _p32), ("s_nslots", _p32),
        ("s_stride", _p32), ("deps", _p32), ("t_mlen", _p32),
        ("gated", _p32), ("ngated", C.c_int64), ("n_gated1", C.c_int32), ("n_up", C.c_int32),
        ("mode", C.c_int32), ("group", C.c_int32), ("split", C.c_int32), ("resident", C.c_int32), ("nunits", C.c_int64), ("nwaves", C.c_int64),
        ("unit0", _p32), ("wave0", _p32), ("u_range", _p64),
        ("res_mat_max", C.c_int64), ("res_vec_max", C.c_int64), ("res_items_max", C.c_int64),
    ]


class H2BError(RuntimeError):
    pass


def _load():
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the H² matvec)")
    lib = C.CDLL(os.fspath(LIB_PATH))
    lib.h2b_abi_version.restype = C.c_int
    if lib.h2b_abi_version() != ABI_VERSION:
        raise RuntimeError(f"{LIB_PATH} has ABI {lib.h2b_abi_version()}, this binding needs {ABI_VERSION}: rebuild it")
    lib.h2b_last_error.restype = C.c_char_p
    # FEM solves (csrc/cg.cu)
    lib.h2b_cg_create.argtypes = [C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_double),
                                  C.POINTER(C.c_void_p)]
    lib.h2b_cg_solve.argtypes = [C.c_void_p, _pd, _pd, C.c_double, C.c_int, C.c_int64, C.POINTER(C.c_int64),
                                 C.POINTER(C.c_double)]
    lib.h2b_cg_solve_dev.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_int, C.c_int64,
                                     C.POINTER(C.c_int64), C.POINTER(C.c_double), C.c_void_p]
    lib.h2b_cg_destroy.argtypes = [C.c_void_p]
    lib.h2b_cg_destroy.restype = None
    lib.h2b_plan_create.argtypes = [C.POINTER(Desc), C.POINTER(Options), C.POINTER(C.c_void_p)]
    lib.h2b_plan_view_get.argtypes = [C.c_void_p, C.POINTER(PlanView)]
    lib.h2b_plan_stats.argtypes = [C.c_void_p, C.POINTER(Stats)]
    lib.h2b_plan_destroy.argtypes = [C.c_void_p]
    lib.h2b_plan_destroy.restype = None
    lib.h2b_create.argtypes = [C.POINTER(Desc), C.POINTER(Options), C.POINTER(C.c_void_p)]
    lib.h2b_matvec_dev.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
    lib.h2b_matvec.argtypes = [C.c_void_p, _pd, _pd, C.c_int64, C.c_int]
    lib.h2b_reset.argtypes = [C.c_void_p]
    lib.h2b_stream_bytes.argtypes = [C.c_void_p]
    lib.h2b_stream_bytes.restype = C.c_int64
    lib.h2b_stats_get.argtypes = [C.c_void_p, C.POINTER(Stats)]
    lib.h2b_destroy.argtypes = [C.c_void_p]
    lib.h2b_destroy.restype = None
    lib.h2b_launch_count.argtypes = [C.c_void_p, C.c_int]
    lib.h2b_launch_count.restype = C.c_int
    lib.h2b_launch_info.argtypes = [C.c_void_p, C.c_int, C.c_int, _p32, _p64, _p64]
    lib.h2b_launch_info.restype = C.c_int
    lib.h2b_launch_times.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p, _pd]
    lib.h2b_launch_times.restype = C.c_int
    lib.h2b_nccl_unique_id.argtypes = [C.c_void_p]
    lib.h2b_plan_phases.argtypes = [C.c_void_p]
    lib.h2b_plan_phase_view.argtypes = [C.c_void_p, C.c_int, C.POINTER(PlanView)]
    lib.h2b_plan_partition.argtypes = [C.c_void_p, _p64, _p64]
    lib.h2b_matvec_phase.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
    lib.h2b_exchange_region.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_void_p), _p64]
    lib.h2b_exchange_copy.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
    lib.h2b_crc64.argtypes = [C.c_void_p, C.c_uint64]
    lib.h2b_crc64.restype = C.c_uint64
    lib.h2b_h2ms_open.argtypes = [C.c_char_p, C.c_int64, C.POINTER(C.c_void_p)]
    lib.h2b_h2ms_desc.argtypes = [C.c_void_p, C.POINTER(Desc)]
    lib.h2b_h2ms_tree.argtypes = [C.c_void_p, _pd, C.POINTER(C.c_uint8)]
    lib.h2b_h2ms_close.argtypes = [C.c_void_p]
    lib.h2b_h2ms_close.restype = None
    lib.h2b_h2ms_write.argtypes = [C.POINTER(Desc), _pd, C.c_char_p]
    for name in ("h2b_h2ms_open", "h2b_h2ms_desc", "h2b_h2ms_tree", "h2b_h2ms_write"):
        getattr(lib, name).restype = C.c_int
    for name in ("h2b_plan_create", "h2b_plan_view_get", "h2b_plan_stats", "h2b_create",
                 "h2b_matvec_dev", "h2b_matvec", "h2b_reset", "h2b_stats_get", "h2b_nccl_unique_id",
                 "h2b_plan_phases", "h2b_plan_phase_view", "h2b_plan_partition", "h2b_matvec_phase",
                 "h2b_exchange_region", "h2b_exchange_copy"):
        getattr(lib, name).restype = C.c_int
    return lib


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = _load()
    return _lib


def check(rc: int, what: str = "h2b") -> None:
    if rc == H2B_OK:
        return
    msg = lib().h2b_last_error().decode(errors="replace")
    if rc == H2B_EINVAL:
        raise ValueError(msg)
    if rc == H2B_EIO:
        from .persist import OperatorIOError
        raise OperatorIOError(msg)
    raise H2BError(f"{what} failed ({rc}): {msg}")


def as_i64_ptr(a: np.ndarray):
    return a.ctypes.data_as(_p64)


def as_d_ptr(a: np.ndarray):
    return a.ctypes.data_as(_pd)


def ptr_array(mats: list) -> tuple:
    """Array of double* from a list of (contiguous float64 ndarray | None)."""
    arr = (_pd * max(1, len(mats)))()
    for i, m in enumerate(mats):
        if m is not None and m.size:
            arr[i] = m.ctypes.data_as(_pd)
    return arr
