"""Closed boundary triangulations for the benchmark configurations and the
per-triangle data the collocation kernel needs.

Only the surface enters the boundary operator: ``CollocationAssembler``
reads the boundary coordinates, the oriented triangles and the solid angles
(/root/reference/pkg/src/strayfield/bem.py:185-191).  The tet-based solid
angle of the reference (mesh.py:97-129) is replaced, for surface-only
meshes, by the equivalent vertex formula

    Psi_i = sum_k theta_k - (n_i - 2) pi,   theta_k = pi - beta_k,

where theta_k is the interior dihedral angle at the k-th edge incident to
vertex i and beta_k the signed bending angle between the outward normals of
the two faces of that edge (the area of the vertex's spherical polygon).

Mesh recipes (BASELINE.json configs; all seeded, all synthetic):

* ``icosphere_surface(r)``  the reference's icosphere shell (mesh.py:287-307)
  with the reference's triangle order, i.e. the boundary of
  ``generate_sphere_mesh(1, r)`` (config 1 uses r = 4);
* ``cube_surface(m)``       [-1,1]^3, m x m quads per face, 2 triangles per
  quad (config 2: m = 130, N = 6 m^2 + 2 = 101 402);
* ``disk_surface(h)``       closed disk, radius 1, thickness 0.05: jittered
  concentric-ring Delaunay faces plus a structured rim (config 3);
* ``sphere_subsample_surface`` random vertex decimation of an icosphere,
  re-triangulated with a convex hull (config 5).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = ["Surface", "make_surface", "solid_angles", "panel_table", "incidence",
           "icosphere_surface", "cube_surface", "disk_surface", "sphere_subsample_surface",
           "PANEL_DOUBLES"]

PANEL_DOUBLES = 34


@dataclass(frozen=True)
class Surface:
    coords: np.ndarray       # (n, 3)
    triangles: np.ndarray    # (T, 3) int64, counter-clockwise seen from outside
    normals: np.ndarray      # (T, 3) unit outward
    areas: np.ndarray        # (T,)
    solid_angles: np.ndarray  # (n,) interior solid angle Psi

    @property
    def n(self) -> int:
        return self.coords.shape[0]

    @property
    def diag(self) -> np.ndarray:
        """D = Psi / 4 pi - 1 (bem.py:191)."""
        return self.solid_angles / (4.0 * math.pi) - 1.0


def _normals_areas(coords, tri):
    p0 = coords[tri[:, 0]]
    nrm = np.cross(coords[tri[:, 1]] - p0, coords[tri[:, 2]] - p0)
    nn = np.linalg.norm(nrm, axis=1)
    if np.any(nn <= 0.0):
        raise ValueError("degenerate triangle with zero area")
    return nrm / nn[:, None], 0.5 * nn


def _check_closed(tri):
    e = np.sort(tri[:, [[0, 1], [1, 2], [2, 0]]].reshape(-1, 2), axis=1)
    _, counts = np.unique(e, axis=0, return_counts=True)
    if not np.all(counts == 2):
        raise ValueError("surface is not closed (dangling or non-manifold edge)")


def solid_angles(coords: np.ndarray, tri: np.ndarray, normals: np.ndarray) -> np.ndarray:
    """Interior solid angle at every vertex of a closed oriented surface."""
    n = coords.shape[0]
    t = tri.shape[0]
    # directed edges u->v of every face, and the face they belong to
    u = tri.reshape(-1)
    v = tri[:, [1, 2, 0]].reshape(-1)
    face = np.repeat(np.arange(t), 3)
    key_fwd = u * n + v
    order = np.argsort(key_fwd, kind="stable")
    sorted_keys = key_fwd[order]
    # partner: the face containing v->u
    key_rev = v * n + u
    pos = np.searchsorted(sorted_keys, key_rev)
    if np.any(pos >= sorted_keys.size) or np.any(sorted_keys[np.minimum(pos, sorted_keys.size - 1)] != key_rev):
        raise ValueError("surface is not closed and consistently oriented")
    partner = face[order[pos]]
    # one record per undirected edge: the directed copy with u < v
    sel = u < v
    uu, vv, f1, f2 = u[sel], v[sel], face[sel], partner[sel]
    n1, n2 = normals[f1], normals[f2]
    e = coords[vv] - coords[uu]
    e /= np.linalg.norm(e, axis=1)[:, None]
    beta = np.arctan2(np.einsum("ij,ij->i", np.cross(n1, n2), e), np.einsum("ij,ij->i", n1, n2))
    theta = math.pi - beta
    psi = np.zeros(n)
    np.add.at(psi, uu, theta)
    np.add.at(psi, vv, theta)
    deg = np.bincount(uu, minlength=n) + np.bincount(vv, minlength=n)
    return psi - (deg - 2) * math.pi


def make_surface(coords: np.ndarray, tri: np.ndarray, psi: np.ndarray | None = None) -> Surface:
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    tri = np.ascontiguousarray(tri, dtype=np.int64)
    _check_closed(tri)
    normals, areas = _normals_areas(coords, tri)
    flux = np.einsum("i,ij->j", areas, normals)
    if np.linalg.norm(flux) > 1e-10 * areas.sum():
        raise ValueError("closed-surface identity violated (orientation)")
    if psi is None:
        psi = solid_angles(coords, tri, normals)
    return Surface(coords=coords, triangles=tri, normals=normals, areas=areas,
                   solid_angles=np.asarray(psi, dtype=np.float64))


def panel_table(s: Surface) -> np.ndarray:
    """(T, 34) per-triangle constants of the analytic kernel (bem.py:67-96):
    vertices, unit normal, in-plane shape-function gradients, gradient . edge
    outward normal table, coplanarity scale, edge lengths."""
    verts = s.coords[s.triangles]                                   # (T,3,3)
    nh = s.normals
    edges = np.stack([verts[:, 1] - verts[:, 0], verts[:, 2] - verts[:, 1],
                      verts[:, 0] - verts[:, 2]], axis=1)
    slen = np.linalg.norm(edges, axis=2)
    m_out = np.cross(edges / slen[:, :, None], nh[:, None, :])
    grads = np.empty_like(verts)
    for i in range(3):
        opp = (i + 1) % 3
        g = np.cross(nh, edges[:, opp])
        grads[:, i] = g / np.einsum("tj,tj->t", g, verts[:, i] - verts[:, opp])[:, None]
    gm = np.einsum("tid,ted->tie", grads, m_out)
    out = np.empty((s.triangles.shape[0], PANEL_DOUBLES))
    out[:, 0:9] = verts.reshape(-1, 9)
    out[:, 9:12] = nh
    out[:, 12:21] = grads.reshape(-1, 9)
    out[:, 21:30] = gm.reshape(-1, 9)
    out[:, 30] = slen.max(axis=1)
    out[:, 31:34] = slen
    return out


def incidence(s: Surface):
    """node -> incident triangles (ascending id) and the node's local vertex."""
    flat = s.triangles.reshape(-1)
    order = np.argsort(flat, kind="stable")       # by node, then by triangle id
    inc_tri = (order // 3).astype(np.int64)
    inc_loc = (order % 3).astype(np.int8)
    inc_ptr = np.zeros(s.n + 1, np.int64)
    inc_ptr[1:] = np.cumsum(np.bincount(flat, minlength=s.n))
    return inc_ptr, inc_tri, inc_loc


# ---------------------------------------------------------------------------
# generators
# ---------------------------------------------------------------------------

_T = (1.0 + math.sqrt(5.0)) / 2.0
_ICO_V = np.array([(-1, _T, 0), (1, _T, 0), (-1, -_T, 0), (1, -_T, 0),
                   (0, -1, _T), (0, 1, _T), (0, -1, -_T), (0, 1, -_T),
                   (_T, 0, -1), (_T, 0, 1), (-_T, 0, -1), (-_T, 0, 1)], dtype=np.float64)
_ICO_F = np.array([(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11),
                   (1, 5, 9), (5, 11, 4), (11, 10, 2), (10, 7, 6), (7, 1, 8),
                   (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9),
                   (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)], dtype=np.int64)


def _unit_rows(v: np.ndarray, exact: bool) -> np.ndarray:
    if exact:
        return np.array([r / np.linalg.norm(r) for r in v]).reshape(v.shape)
    return v / np.linalg.norm(v, axis=1)[:, None]


def _icosphere(level: int):
    """Vectorised midpoint subdivision.  Vertex numbering equals the
    reference's dict-based construction (mesh.py:287-307): new midpoints are
    numbered in order of first appearance while sweeping faces (i,j),(j,k),(k,i)."""
    exact = level <= 6   # per-vector norms: bit-identical to the reference's loop
    verts = _unit_rows(_ICO_V, exact)
    faces = _ICO_F.copy()
    for _ in range(level):
        nv = verts.shape[0]
        e = np.stack([faces[:, [0, 1]], faces[:, [1, 2]], faces[:, [2, 0]]], axis=1).reshape(-1, 2)
        key = np.minimum(e[:, 0], e[:, 1]) * (nv + 1) + np.maximum(e[:, 0], e[:, 1])
        uniq, first, inv = np.unique(key, return_index=True, return_inverse=True)
        # number midpoints by first appearance in the sweep
        rank = np.empty(uniq.size, np.int64)
        rank[np.argsort(first, kind="stable")] = np.arange(uniq.size)
        mid_id = nv + rank[inv].reshape(-1, 3)
        a = np.minimum(e[:, 0], e[:, 1])[first]
        b = np.maximum(e[:, 0], e[:, 1])[first]
        # reference: v = verts[i] + verts[j] with (i, j) as first met (order of the sum is exact either way)
        mids = _unit_rows(verts[a] + verts[b], exact)
        new_verts = np.empty((nv + uniq.size, 3))
        new_verts[:nv] = verts
        new_verts[nv + rank] = mids
        i, j, k = faces[:, 0], faces[:, 1], faces[:, 2]
        ij, jk, ki = mid_id[:, 0], mid_id[:, 1], mid_id[:, 2]
        faces = np.stack([np.stack([i, ij, ki], 1), np.stack([j, jk, ij], 1),
                          np.stack([k, ki, jk], 1), np.stack([ij, jk, ki], 1)], axis=1).reshape(-1, 3)
        verts = new_verts
    return verts, faces


def icosphere_surface(level: int, radius: float = 1.0) -> Surface:
    verts, faces = _icosphere(level)
    # the reference's extract_surface returns faces ordered by sorted vertex key
    order = np.lexsort(np.sort(faces, axis=1).T[::-1])
    return make_surface(verts * radius, faces[order])


def cube_surface(m: int = 130) -> Surface:
    """Surface of [-1,1]^3 with m x m quads per face, 2 triangles per quad,
    nodes numbered lexicographically by lattice index (i, j, k)."""
    g = np.arange(m + 1)
    I, J, K = np.meshgrid(g, g, g, indexing="ij")
    on = (I == 0) | (I == m) | (J == 0) | (J == m) | (K == 0) | (K == m)
    lat = np.stack([I[on], J[on], K[on]], axis=1)          # lexicographic order
    idx = -np.ones((m + 1,) * 3, np.int64)
    idx[lat[:, 0], lat[:, 1], lat[:, 2]] = np.arange(lat.shape[0])
    coords = -1.0 + 2.0 * lat / m
    tris = []
    a = np.arange(m)
    A, B = np.meshgrid(a, a, indexing="ij")
    A, B = A.ravel(), B.ravel()
    for axis in range(3):
        u, w = [d for d in range(3) if d != axis]
        for side, sgn in ((0, -1.0), (m, 1.0)):
            def node(da, db):
                ijk = [None, None, None]
                ijk[axis] = np.full(A.shape, side)
                ijk[u] = A + da
                ijk[w] = B + db
                return idx[ijk[0], ijk[1], ijk[2]]
            q0, q1, q2, q3 = node(0, 0), node(1, 0), node(1, 1), node(0, 1)
            t1 = np.stack([q0, q1, q2], 1)
            t2 = np.stack([q0, q2, q3], 1)
            t = np.concatenate([t1, t2])
            # orient outward: (e_u x e_w) has the sign of +axis for cyclic (u, w)
            cyc = ((u - axis) % 3) == 1
            if (sgn > 0) != cyc:
                t = t[:, [0, 2, 1]]
            tris.append(t)
    return make_surface(coords, np.concatenate(tris))


def disk_surface(h: float = 0.0025, radius: float = 1.0, thickness: float = 0.05,
                 seed: int = 1234, jitter: float = 0.2) -> Surface:
    """Closed thin disk: jittered concentric-ring Delaunay faces (z = +-t/2)
    sharing an unjittered rim ring with a structured rim band."""
    from scipy.spatial import Delaunay
    rng = np.random.default_rng(seed)
    n_theta = int(round(2.0 * math.pi * radius / h))
    n_rings = int(round(thickness / h)) + 1
    th = 2.0 * math.pi * np.arange(n_theta) / n_theta
    rim_xy = np.stack([radius * np.cos(th), radius * np.sin(th)], 1)
    # interior face points: centre + concentric rings, jittered
    pts = [np.zeros((1, 2))]
    n_int = int(round(radius / h))
    for i in range(1, n_int):
        r = i * h
        k = max(3, int(round(2.0 * math.pi * r / h)))
        phi = 2.0 * math.pi * (np.arange(k) + 0.5 * (i % 2)) / k
        pts.append(np.stack([r * np.cos(phi), r * np.sin(phi)], 1))
    inner = np.concatenate(pts)
    faces_xy = []
    for _ in range(2):
        faces_xy.append(inner + rng.uniform(-jitter * h, jitter * h, inner.shape))
    z_levels = np.linspace(-thickness / 2, thickness / 2, n_rings)
    # node numbering: bottom interior, top interior, rim rings bottom -> top
    nb = inner.shape[0]
    coords = [np.column_stack([faces_xy[0], np.full(nb, z_levels[0])]),
              np.column_stack([faces_xy[1], np.full(nb, z_levels[-1])])]
    for z in z_levels:
        coords.append(np.column_stack([rim_xy, np.full(n_theta, z)]))
    coords = np.concatenate(coords)
    rim0 = 2 * nb
    tris = []
    for f, (sgn, ring) in enumerate(((-1.0, 0), (1.0, n_rings - 1))):
        xy = np.concatenate([faces_xy[f], rim_xy])
        ids = np.concatenate([np.arange(nb) + f * nb, rim0 + ring * n_theta + np.arange(n_theta)])
        tri = Delaunay(xy).simplices
        p = xy[tri]
        cr = (p[:, 1, 0] - p[:, 0, 0]) * (p[:, 2, 1] - p[:, 0, 1]) - (p[:, 1, 1] - p[:, 0, 1]) * (p[:, 2, 0] - p[:, 0, 0])
        flip = (cr > 0) != (sgn > 0)
        tri[flip] = tri[flip][:, [0, 2, 1]]
        tris.append(ids[tri])
    j = np.arange(n_theta)
    jn = (j + 1) % n_theta
    for ring in range(n_rings - 1):
        b0 = rim0 + ring * n_theta
        b1 = b0 + n_theta
        # quad (j, jn) x (ring, ring+1); outward = radial
        tris.append(np.stack([b0 + j, b0 + jn, b1 + jn], 1))
        tris.append(np.stack([b0 + j, b1 + jn, b1 + j], 1))
    return make_surface(coords, np.concatenate(tris))


def sphere_subsample_surface(level: int = 10, npts: int = 4_194_304, seed: int = 1234,
                             radius: float = 1.0) -> Surface:
    """Seeded random vertex decimation of an icosphere, re-triangulated by
    its convex hull (all points lie on the sphere, so all are hull vertices)."""
    from scipy.spatial import ConvexHull
    verts, _ = _icosphere(level)
    rng = np.random.default_rng(seed)
    keep = np.sort(rng.choice(verts.shape[0], npts, replace=False))
    pts = verts[keep] * radius
    hull = ConvexHull(pts)
    tri = hull.simplices.astype(np.int64)
    p0 = pts[tri[:, 0]]
    nrm = np.cross(pts[tri[:, 1]] - p0, pts[tri[:, 2]] - p0)
    inward = np.einsum("ij,ij->i", nrm, p0) < 0
    tri[inward] = tri[inward][:, [0, 2, 1]]
    return make_surface(pts, tri)
