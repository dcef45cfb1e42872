"""Operator files: the reference's "H2MS" v1 format, natively.

Mirrors ``strayfield.hmatrix.persist`` (hmatrix/persist.py:22-199): the same
byte layout (little-endian magic "H2MS", u32 version 1, u64 N, the
permutation, the preorder cluster tree, both sides' leaf bases and
transfers, coupling and near-field blocks, trailing CRC-64/XZ of every
preceding byte), the same public functions and the same ``OperatorIOError``
messages.  Reading, checking and writing run in libh2b (csrc/h2ms.cpp): the
checksum uses every host core, and :func:`load_device_operator` takes a file
straight into the GPU layout without building Python matrices.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from . import _native as nat
from .cluster import Cluster, ClusterTree, tree_arrays
from .h2 import DeviceOperator, H2Matrix, describe

__all__ = ["OperatorIOError", "crc64", "save_h2", "load_h2", "load_device_operator", "H2MSFile"]


class OperatorIOError(IOError):
    """Corrupt or incompatible compressed-operator file (errors.py:18-19)."""


def crc64(data) -> int:
    """CRC-64/XZ of ``data`` (persist.py:34-38)."""
    buf = memoryview(data).cast("B") if not isinstance(data, (bytes, bytearray)) else data
    arr = np.frombuffer(buf, dtype=np.uint8)
    return int(nat.lib().h2b_crc64(arr.ctypes.data_as(C.c_void_p), arr.size))


def save_h2(op, path) -> None:
    """Serialize an H² operator (persist.py:117-135), byte-identical to the
    reference's writer."""
    h = describe(op)
    ta = tree_arrays(op.tree)
    bbox = np.ascontiguousarray(np.hstack([ta["cl_bbox_min"], ta["cl_bbox_max"]]), dtype=np.float64)
    nat.check(nat.lib().h2b_h2ms_write(C.byref(h.desc), nat.as_d_ptr(bbox), os.fsencode(str(path))),
              "h2b_h2ms_write")


class H2MSFile:
    """An opened, verified operator file held by libh2b (``h2b_h2ms``)."""

    def __init__(self, path, expected_n: int | None = None):
        self._lib = nat.lib()
        h = C.c_void_p()
        nat.check(self._lib.h2b_h2ms_open(os.fsencode(str(path)), -1 if expected_n is None else int(expected_n),
                                          C.byref(h)), "h2b_h2ms_open")
        self._h = h
        self.desc = nat.Desc()
        nat.check(self._lib.h2b_h2ms_desc(self._h, C.byref(self.desc)), "h2b_h2ms_desc")

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.h2b_h2ms_close(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def to_h2matrix(self) -> H2Matrix:
        d = self.desc
        n, nc = int(d.n), int(d.nclusters)

        def arr(ptr, count, dtype=np.int64):
            return np.ctypeslib.as_array(ptr, shape=(count,)).astype(dtype, copy=True) if count else \
                np.zeros(0, dtype)

        def mat(ptr, r, c):
            if r * c == 0 or not ptr:
                return np.zeros((r, c))
            return np.ctypeslib.as_array(ptr, shape=(r * c,)).reshape(r, c).copy()

        perm = arr(d.perm, n)
        start, end = arr(d.cl_start, nc), arr(d.cl_end, nc)
        child = arr(d.cl_child, 2 * nc).reshape(nc, 2)
        k_row, k_col = arr(d.k_row, nc), arr(d.k_col, nc)
        bbox = np.zeros((nc, 6))
        leaf = np.zeros(nc, np.uint8)
        nat.check(self._lib.h2b_h2ms_tree(self._h, nat.as_d_ptr(bbox),
                                          leaf.ctypes.data_as(C.POINTER(C.c_uint8))), "h2b_h2ms_tree")
        clusters = [Cluster(int(start[i]), int(end[i]), bbox[i, :3].copy(), bbox[i, 3:].copy(), cid=i)
                    for i in range(nc)]
        for i in range(nc):
            if child[i, 0] >= 0:
                clusters[i].children = (clusters[int(child[i, 0])], clusters[int(child[i, 1])])
        tree = ClusterTree(root=clusters[0], perm=perm, clusters=clusters)
        op = H2Matrix(tree=tree, n=n)
        size = end - start
        for i in range(nc):
            if child[i, 0] < 0:
                op.row_basis[i] = mat(d.row_basis[i], size[i], k_row[i])
                op.col_basis[i] = mat(d.col_basis[i], size[i], k_col[i])
            else:
                for ch in child[i]:
                    op.row_transfer[int(ch)] = mat(d.row_transfer[ch], k_row[ch], k_row[i])
                    op.col_transfer[int(ch)] = mat(d.col_transfer[ch], k_col[ch], k_col[i])
        cp_row, cp_col = arr(d.cp_row, d.ncoupling), arr(d.cp_col, d.ncoupling)
        for b in range(int(d.ncoupling)):
            t, s = int(cp_row[b]), int(cp_col[b])
            op.coupling.append((t, s, mat(d.cp_data[b], k_row[t], k_col[s])))
        nr_row, nr_col = arr(d.nr_row, d.nnear), arr(d.nr_col, d.nnear)
        for b in range(int(d.nnear)):
            t, s = int(nr_row[b]), int(nr_col[b])
            op.near.append((t, s, mat(d.nr_data[b], size[t], size[s])))
        return op


def load_h2(path, expected_n: int | None = None) -> H2Matrix:
    """Read an operator back (persist.py:138-199); raises OperatorIOError on a
    bad magic number, unsupported version, truncation, checksum mismatch, or
    when the stored node count disagrees with ``expected_n``."""
    with H2MSFile(path, expected_n) as f:
        return f.to_h2matrix()


def load_device_operator(path, expected_n: int | None = None, **options) -> DeviceOperator:
    """Operator file -> GPU operator, with no Python matrices in between."""
    with H2MSFile(path, expected_n) as f:
        return DeviceOperator.from_desc(f.desc, **options)
