"""Cluster tree data model consumed by the H² matvec.

Mirrors the reference's ``Cluster`` / ``ClusterTree``
(/root/reference/pkg/src/strayfield/hmatrix/cluster.py:13-59): a binary tree
of contiguous index ranges under a permutation, numbered in preorder.  Only
the fields the matvec and the flattener read are required; the reference's
own objects are accepted everywhere these are (duck typing), so the GPU path
is a drop-in for operators built by the reference.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["Cluster", "ClusterTree", "tree_arrays", "tree_from_arrays"]


@dataclass(eq=False)
class Cluster:
    """Contiguous index range ``[start, end)`` of tree positions
    (cluster.py:13-37)."""

    start: int
    end: int
    bbox_min: np.ndarray
    bbox_max: np.ndarray
    children: tuple["Cluster", ...] = ()
    cid: int = -1

    @property
    def size(self) -> int:
        return self.end - self.start

    @property
    def is_leaf(self) -> bool:
        return not self.children

    def diameter(self) -> float:
        return float(np.linalg.norm(self.bbox_max - self.bbox_min))


@dataclass(eq=False)
class ClusterTree:
    """``perm[pos]`` is the original node index at tree position ``pos``;
    ``clusters`` is the preorder list (cluster.py:40-59)."""

    root: Cluster
    perm: np.ndarray
    clusters: list[Cluster] = field(default_factory=list)

    @property
    def n_points(self) -> int:
        return self.perm.shape[0]

    def indices(self, cluster: Cluster) -> np.ndarray:
        return self.perm[cluster.start:cluster.end]


def tree_arrays(tree) -> dict[str, np.ndarray]:
    """Structure-of-arrays form of a (reference or mirror) cluster tree."""
    cl = tree.clusters
    nc = len(cl)
    start = np.empty(nc, np.int64)
    end = np.empty(nc, np.int64)
    child = np.full((nc, 2), -1, np.int64)
    bmin = np.empty((nc, 3))
    bmax = np.empty((nc, 3))
    for i, c in enumerate(cl):
        if c.cid != i:
            raise ValueError("cluster list is not in preorder-id order")
        start[i] = c.start
        end[i] = c.end
        bmin[i] = c.bbox_min
        bmax[i] = c.bbox_max
        if c.children:
            if len(c.children) != 2:
                raise ValueError("cluster tree must be binary")
            child[i] = [c.children[0].cid, c.children[1].cid]
    return {
        "perm": np.ascontiguousarray(tree.perm, dtype=np.int64),
        "cl_start": start,
        "cl_end": end,
        "cl_child": child,
        "cl_bbox_min": bmin,
        "cl_bbox_max": bmax,
    }


def tree_from_arrays(a: dict[str, np.ndarray]) -> ClusterTree:
    """Inverse of :func:`tree_arrays` (preorder ids preserved)."""
    start, end, child = a["cl_start"], a["cl_end"], a["cl_child"]
    bmin, bmax = a["cl_bbox_min"], a["cl_bbox_max"]
    nc = start.shape[0]
    clusters = [Cluster(int(start[i]), int(end[i]), bmin[i].copy(), bmax[i].copy(), cid=i)
                for i in range(nc)]
    for i in range(nc):
        if child[i, 0] >= 0:
            clusters[i].children = (clusters[int(child[i, 0])], clusters[int(child[i, 1])])
    return ClusterTree(root=clusters[0], perm=np.asarray(a["perm"], np.int64).copy(),
                       clusters=clusters)
