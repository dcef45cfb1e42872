"""Compact numpy (.npz) container for an H² operator.

Used for the committed golden fixtures (operators built by the reference in
the build container) and for caching operators built on the GPU box.  This
is not the reference's "H2MS" format (persist.py:22-199); it stores the same
fields (tree, per-side bases/transfers, coupling and near-field lists) as a
few flat arrays so that loading is a handful of numpy reads.
"""

from __future__ import annotations

import numpy as np

from .cluster import tree_arrays, tree_from_arrays
from .h2 import H2Matrix

__all__ = ["h2_to_arrays", "h2_from_arrays", "save_npz", "load_npz"]


def _pack_dict(prefix: str, d: dict) -> dict:
    ids = np.array(sorted(d), dtype=np.int64)
    shapes = np.array([d[i].shape for i in ids], dtype=np.int64).reshape(-1, 2)
    data = (np.concatenate([np.ascontiguousarray(d[i], np.float64).ravel() for i in ids])
            if len(ids) else np.zeros(0))
    return {f"{prefix}_ids": ids, f"{prefix}_shapes": shapes, f"{prefix}_data": data}


def _unpack_dict(a, prefix: str) -> dict:
    ids, shapes, data = a[f"{prefix}_ids"], a[f"{prefix}_shapes"], a[f"{prefix}_data"]
    out = {}
    off = 0
    for i, (r, c) in zip(ids, shapes):
        out[int(i)] = data[off: off + r * c].reshape(r, c)
        off += r * c
    return out


def _pack_list(prefix: str, blocks: list) -> dict:
    rows = np.array([b[0] for b in blocks], dtype=np.int64)
    cols = np.array([b[1] for b in blocks], dtype=np.int64)
    shapes = np.array([b[2].shape for b in blocks], dtype=np.int64).reshape(-1, 2)
    data = (np.concatenate([np.ascontiguousarray(b[2], np.float64).ravel() for b in blocks])
            if blocks else np.zeros(0))
    return {f"{prefix}_row": rows, f"{prefix}_col": cols, f"{prefix}_shapes": shapes,
            f"{prefix}_data": data}


def _unpack_list(a, prefix: str) -> list:
    rows, cols, shapes, data = (a[f"{prefix}_row"], a[f"{prefix}_col"], a[f"{prefix}_shapes"],
                                a[f"{prefix}_data"])
    out = []
    off = 0
    for r, c, (nr, nc) in zip(rows, cols, shapes):
        out.append((int(r), int(c), data[off: off + nr * nc].reshape(nr, nc)))
        off += nr * nc
    return out


def h2_to_arrays(op) -> dict:
    a = {"n": np.array(op.n, dtype=np.int64)}
    a.update(tree_arrays(op.tree))
    a.update(_pack_dict("rb", op.row_basis))
    a.update(_pack_dict("cb", op.col_basis))
    a.update(_pack_dict("rt", op.row_transfer))
    a.update(_pack_dict("ct", op.col_transfer))
    a.update(_pack_list("cp", op.coupling))
    a.update(_pack_list("nr", op.near))
    return a


def h2_from_arrays(a) -> H2Matrix:
    tree = tree_from_arrays({k: a[k] for k in ("perm", "cl_start", "cl_end", "cl_child",
                                               "cl_bbox_min", "cl_bbox_max")})
    return H2Matrix(tree=tree, n=int(a["n"]),
                    row_basis=_unpack_dict(a, "rb"), row_transfer=_unpack_dict(a, "rt"),
                    col_basis=_unpack_dict(a, "cb"), col_transfer=_unpack_dict(a, "ct"),
                    coupling=_unpack_list(a, "cp"), near=_unpack_list(a, "nr"))


def save_npz(op, path, **extra) -> None:
    a = h2_to_arrays(op)
    for k, v in extra.items():
        a["x_" + k] = np.asarray(v)
    np.savez_compressed(path, **a)


def load_npz(path) -> tuple[H2Matrix, dict]:
    """Returns (operator, extras) where extras holds every ``x_*`` array
    saved alongside (without the prefix)."""
    with np.load(path) as z:
        a = {k: z[k] for k in z.files}
    extras = {k[2:]: v for k, v in a.items() if k.startswith("x_")}
    return h2_from_arrays(a), extras
