"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container only (it imports /root/reference/pkg/src, which
does not exist on the GPU box):

    python tests/golden/make_golden.py

For each case it builds the H² operator with the reference's own
``hmatrix.assemble_operator`` (hmatrix/__init__.py:31-44), stores it in the
compact npz container (paper_1811_05731_b200/io.py), and records the
reference's outputs on seeded inputs:

* ``y_full``  reference ``h2_matvec(op, x)``                (h2.py:186-244)
* ``y_near``  reference h2_matvec of ``replace(op, coupling=[])``
* ``y_far``   reference h2_matvec of ``replace(op, near=[])``
* ``y_dense`` reference dense operator ``assemble_dense(mesh) @ x``
  (bem.py:264-274), for the H²-vs-dense accuracy checks of the reference's
  own tests (test_hmatrix.py:272-278, test_acceptance.py:80-100)
* config 1 also stores the uniformly-magnetized-sphere pipeline result
  ``compute_demag`` (pipeline.py:46-63) and a hash of the tet mesh, so the
  GPU energy test can rebuild the mesh with the oracle's restated generator
  and check it is the reference's mesh.
"""

from __future__ import annotations

import dataclasses
import hashlib
import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(REF))
sys.path.insert(0, str(ROOT))

from strayfield import bem, pipeline  # noqa: E402
from strayfield import hmatrix as hm  # noqa: E402
from strayfield import mesh as meshmod  # noqa: E402
from strayfield.hmatrix.h2 import h2_matvec as ref_h2_matvec  # noqa: E402

from paper_1811_05731_b200.io import save_npz  # noqa: E402


def mesh_hash(mesh) -> str:
    h = hashlib.sha256()
    for a in (mesh.nodes, mesh.tets, mesh.boundary_nodes, mesh.surface.triangles):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


CASES = {
    # name: (mesh factory, CompressionConfig kwargs, dense?, energy?)
    "config1_sphere4": (lambda: meshmod.generate_sphere_mesh(1.0, 4),
                        dict(leaf_size=32, eta=2.0, cheb_order=4), True, True),
    "sphere3_l32_eta2_o4": (lambda: meshmod.generate_sphere_mesh(1.0, 3),
                            dict(leaf_size=32, eta=2.0, cheb_order=4), True, False),
    "sphere2_default": (lambda: meshmod.generate_sphere_mesh(1.0, 2), {}, True, False),
    "torus_32_16_4_default": (lambda: meshmod.generate_torus_mesh(2.0, 1.0, 32, 16, 4), {}, True, False),
    "prism_20_40_2_default": (lambda: meshmod.generate_prism_mesh(10.0, 20.0, 1.0, 20, 40, 2), {}, True, False),
}


def make(name: str) -> None:
    factory, cfg_kw, want_dense, want_energy = CASES[name]
    t0 = time.perf_counter()
    mesh = factory()
    cfg = hm.CompressionConfig(**cfg_kw)
    op = hm.assemble_operator(mesh, "h2", cfg)
    h2 = op.payload
    t_build = time.perf_counter() - t0
    n = h2.n
    rng = np.random.default_rng(1234)
    xs = [rng.standard_normal(n) for _ in range(3)]
    coords = mesh.boundary_coords()
    xs.append(np.ones(n))
    if name.startswith(("config1", "sphere")):
        xs.append(coords[:, 2] / 3.0)          # u1 = z/3 test vector (BASELINE.json)
    for j in rng.choice(n, 3, replace=False):
        e = np.zeros(n)
        e[j] = 1.0
        xs.append(e)
    X = np.stack(xs, axis=1)
    y_full = np.stack([ref_h2_matvec(h2, X[:, i]) for i in range(X.shape[1])], axis=1)
    near_op = dataclasses.replace(h2, coupling=[])
    far_op = dataclasses.replace(h2, near=[])
    y_near = np.stack([ref_h2_matvec(near_op, X[:, i]) for i in range(X.shape[1])], axis=1)
    y_far = np.stack([ref_h2_matvec(far_op, X[:, i]) for i in range(X.shape[1])], axis=1)
    extra = dict(X=X, y_full=y_full, y_near=y_near, y_far=y_far,
                 storage_bytes=np.array(h2.storage_bytes()),
                 config=np.array([cfg.leaf_size, cfg.eta, cfg.cheb_order, cfg.eps, cfg.eps_rec]),
                 boundary_coords=coords,
                 diag=mesh.boundary_solid_angles() / (4.0 * np.pi) - 1.0,
                 surface_triangles=mesh.surface.triangles)
    if want_dense:
        dense = bem.assemble_dense(mesh)
        extra["y_dense"] = dense.payload @ X
        extra["dense_norm"] = np.array(np.linalg.norm(dense.payload))
        # columns of the dense operator at the unit vectors (test_unit_vector_columns)
    if want_energy:
        m = pipeline.magnetization_preset(mesh, "uniform-z")
        res = pipeline.compute_demag(mesh, m, op)
        extra["energy_e_d_over_kd"] = np.array(res.e_d_over_kd)
        extra["energy_u1_boundary"] = res.u1[mesh.boundary_nodes]
        extra["energy_u2_boundary"] = res.u2[mesh.boundary_nodes]
        extra["energy_iterations"] = np.array([res.u1_iterations, res.u2_iterations])
        extra["mesh_sha256"] = np.frombuffer(mesh_hash(mesh).encode(), dtype=np.uint8)
        extra["mesh_counts"] = np.array([mesh.n_nodes, mesh.n_tets, mesh.n_boundary])
    path = HERE / f"{name}.npz"
    save_npz(h2, path, **extra)
    ncp, nnr = len(h2.coupling), len(h2.near)
    print(f"{name}: n={n} clusters={len(h2.tree.clusters)} coupling={ncp} near={nnr} "
          f"bytes={h2.storage_bytes()} build={t_build:.1f}s file={path.stat().st_size/1e6:.2f}MB"
          + (f" e_d/K_d={extra['energy_e_d_over_kd']!r}" if want_energy else ""), flush=True)


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for nm in names:
        make(nm)
