"""Restated sphere tet-mesh generator — TEST INFRASTRUCTURE ONLY.

Rebuilds the reference's ``generate_sphere_mesh(radius, refinement)``
(/root/reference/pkg/src/strayfield/mesh.py:334-367: icosphere shells,
radial layers, prisms split into three tets by coning the lowest vertex,
mesh.py:287-331) and the oriented boundary extraction
(mesh.py:135-179) so the energy check can run on the GPU box, where the
reference is absent.  The golden fixture stores a SHA-256 of the reference's
mesh; tests assert this restatement reproduces it bit for bit.
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass

import numpy as np

__all__ = ["SphereMesh", "generate_sphere_mesh", "mesh_hash"]

_T = (1.0 + math.sqrt(5.0)) / 2.0
_V0 = np.array([(-1, _T, 0), (1, _T, 0), (-1, -_T, 0), (1, -_T, 0),
                (0, -1, _T), (0, 1, _T), (0, -1, -_T), (0, 1, -_T),
                (_T, 0, -1), (_T, 0, 1), (-_T, 0, -1), (-_T, 0, 1)], dtype=np.float64)
_F0 = np.array([(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11),
                (1, 5, 9), (5, 11, 4), (11, 10, 2), (10, 7, 6), (7, 1, 8),
                (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9),
                (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)], dtype=np.int64)
_FACES_OF_TET = np.array([[1, 2, 3], [0, 3, 2], [0, 1, 3], [0, 2, 1]])


@dataclass(frozen=True)
class SphereMesh:
    nodes: np.ndarray
    tets: np.ndarray
    boundary_nodes: np.ndarray
    triangles: np.ndarray   # boundary-local, outward

    @property
    def n_nodes(self) -> int:
        return self.nodes.shape[0]

    @property
    def n_boundary(self) -> int:
        return self.boundary_nodes.shape[0]


def _shell(refinement: int):
    verts = [v / np.linalg.norm(v) for v in _V0]
    faces = [tuple(f) for f in _F0.tolist()]
    for _ in range(refinement):
        cache: dict = {}

        def midpoint(a, b):
            key = (a, b) if a < b else (b, a)
            idx = cache.get(key)
            if idx is None:
                v = verts[a] + verts[b]
                verts.append(v / np.linalg.norm(v))
                idx = cache[key] = len(verts) - 1
            return idx

        nxt = []
        for a, b, c in faces:
            ab, bc, ca = midpoint(a, b), midpoint(b, c), midpoint(c, a)
            nxt.extend([(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)])
        faces = nxt
    return np.array(verts), np.array(faces, dtype=np.int64)


def _quad_split(q):
    m = min(range(4), key=lambda i: q[i])
    return ((q[m], q[(m + 1) % 4], q[(m + 2) % 4]), (q[m], q[(m + 2) % 4], q[(m + 3) % 4]))


def _prism_tets(bot, top):
    apex = min(bot + top)
    faces = [bot, top]
    for i in range(3):
        j = (i + 1) % 3
        faces.extend(_quad_split((bot[i], bot[j], top[j], top[i])))
    return [(apex,) + tuple(f) for f in faces if apex not in f]


def generate_sphere_mesh(radius: float, refinement: int) -> SphereMesh:
    shell, faces = _shell(refinement)
    nv = shell.shape[0]
    layers = 2 ** refinement
    nodes = np.empty((1 + layers * nv, 3))
    nodes[0] = 0.0
    for layer in range(1, layers + 1):
        nodes[1 + (layer - 1) * nv: 1 + layer * nv] = shell * (radius * layer / layers)

    def lid(layer, v):
        return 1 + (layer - 1) * nv + v

    tets = [(0, lid(1, i), lid(1, j), lid(1, k)) for i, j, k in faces]
    for layer in range(1, layers):
        for i, j, k in faces:
            tets.extend(_prism_tets((lid(layer, i), lid(layer, j), lid(layer, k)),
                                    (lid(layer + 1, i), lid(layer + 1, j), lid(layer + 1, k))))
    nodes = np.ascontiguousarray(nodes, dtype=np.float64)
    tets = np.ascontiguousarray(np.array(tets, dtype=np.int64))
    # orientation: positive signed volume
    p = nodes[tets]
    vol = np.einsum("ij,ij->i", p[:, 1] - p[:, 0], np.cross(p[:, 2] - p[:, 0], p[:, 3] - p[:, 0])) / 6.0
    neg = vol < 0.0
    tets[neg] = tets[neg][:, [0, 1, 3, 2]]
    # boundary faces: appear in exactly one tet; orient away from the 4th vertex
    flat = tets[:, _FACES_OF_TET].reshape(-1, 3)
    _, first, counts = np.unique(np.sort(flat, axis=1), axis=0, return_index=True, return_counts=True)
    pos = first[counts == 1]
    tri = flat[pos]
    opp = tets[pos // 4, pos % 4]
    p0 = nodes[tri[:, 0]]
    nrm = np.cross(nodes[tri[:, 1]] - p0, nodes[tri[:, 2]] - p0)
    inward = np.einsum("ij,ij->i", nrm, nodes[opp] - p0) > 0
    tri[inward] = tri[inward][:, [0, 2, 1]]
    bnodes = np.unique(tri)
    local = np.full(nodes.shape[0], -1, dtype=np.int64)
    local[bnodes] = np.arange(bnodes.size)
    return SphereMesh(nodes=nodes, tets=tets, boundary_nodes=bnodes, triangles=local[tri])


def mesh_hash(mesh: SphereMesh) -> str:
    h = hashlib.sha256()
    for a in (mesh.nodes, mesh.tets, mesh.boundary_nodes, mesh.triangles):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()
