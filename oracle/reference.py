"""The UNMODIFIED reference, imported from ``baseline/_ref`` — TEST AND
BENCH INFRASTRUCTURE ONLY.

``baseline/_ref`` is the reference package installed by pip from
``/root/reference/pkg`` (git-ignored, shipped to the GPU box by gpurun; see
DESIGN.md §3).  Its tests (``/root/reference/pkg/tests``) are copied next
to it as ``baseline/_ref/tests`` by ``tools/vendor_reference.sh``.  Nothing in
``paper_1811_05731_b200/`` imports this module: it is the checker (tests) and
the reference arm of ``bench.py``, never the product path.

* :func:`strayfield` imports the reference package from ``baseline/_ref``.
* :func:`to_reference` wraps an operator held by this repo (the mirror
  ``H2Matrix``) into the reference's own ``H2Matrix``/``ClusterTree``/
  ``Cluster`` objects (strayfield/hmatrix/h2.py:23-42, cluster.py:13-59),
  sharing the matrices (no copies), so ``strayfield.hmatrix.h2.h2_matvec``
  (h2.py:186-244) runs on it unchanged.
* :func:`structure_twin` builds, on the host CPU only (no GPU, no native
  library), an operator with exactly the structure of a workload's operator
  — the same surface, cluster tree, block partition and per-cluster ranks,
  hence the same block shapes and ``storage_bytes()`` — with seeded N(0,1)
  entries.  The reference matvec's cost depends on those shapes only
  (one numpy GEMV per block), so this is how the reference arm times the
  reference on the full workload without rebuilding the operator on the GPU.
"""

from __future__ import annotations

import importlib
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
REF_DIR = ROOT / "baseline" / "_ref"

__all__ = ["REF_DIR", "available", "strayfield", "to_reference", "reference_h2_matvec", "structure_twin",
           "rank_fixture_path"]


def available() -> bool:
    return (REF_DIR / "strayfield" / "hmatrix" / "h2.py").exists()


def strayfield():
    """The reference package (``import strayfield`` from baseline/_ref)."""
    if not available():
        raise RuntimeError(f"{REF_DIR} is missing: run tools/vendor_reference.sh")
    p = str(REF_DIR)
    if p not in sys.path:
        sys.path.insert(0, p)
    mod = importlib.import_module("strayfield")   # a namespace package in the reference (no __init__)
    where = [str(Path(q).resolve()) for q in getattr(mod, "__path__", [])]
    if not where or not all(w.startswith(str(REF_DIR.resolve())) for w in where):
        raise RuntimeError(f"strayfield imported from {where}, not {REF_DIR}")
    importlib.import_module("strayfield.hmatrix")
    return mod


def to_reference(op):
    """The reference's H2Matrix over the same matrices as ``op``."""
    sf = strayfield()
    cl_mod = sys.modules["strayfield.hmatrix.cluster"]
    h2_mod = sys.modules["strayfield.hmatrix.h2"]
    src = op.tree.clusters
    clusters = [cl_mod.Cluster(int(c.start), int(c.end), np.asarray(c.bbox_min), np.asarray(c.bbox_max),
                               cid=int(c.cid)) for c in src]
    for c in src:
        if c.children:
            clusters[c.cid].children = tuple(clusters[ch.cid] for ch in c.children)
    tree = cl_mod.ClusterTree(root=clusters[0], perm=np.asarray(op.tree.perm, np.int64), clusters=clusters)
    return h2_mod.H2Matrix(tree=tree, n=int(op.n), row_basis=dict(op.row_basis), row_transfer=dict(op.row_transfer),
                           col_basis=dict(op.col_basis), col_transfer=dict(op.col_transfer),
                           coupling=list(op.coupling), near=list(op.near))


def reference_h2_matvec():
    """``strayfield.hmatrix.h2.h2_matvec`` as shipped (h2.py:186-244)."""
    strayfield()
    return sys.modules["strayfield.hmatrix.h2"].h2_matvec


def rank_fixture_path(name: str) -> Path:
    return ROOT / "tests" / "golden" / f"{name}_structure.npz"


def structure_twin(name: str, seed: int = 7, log=lambda m: None):
    """(mirror H2Matrix, info): the workload's operator structure from the
    committed fixture ``tests/golden/<name>_structure.npz`` (per-cluster
    ranks of the operator built on the GPU box by tools/structure_fixture.py,
    and its storage_bytes), the tree and block partition recomputed on the
    host, entries seeded N(0,1)."""
    import time
    from paper_1811_05731_b200.assembly.hbuild import build_cluster_tree, leaf_block_list
    from paper_1811_05731_b200.h2 import H2Matrix
    from paper_1811_05731_b200.workloads import WORKLOADS
    fx = np.load(rank_fixture_path(name))
    w = WORKLOADS[name]
    t0 = time.perf_counter()
    surf = w["surface"]()
    tree = build_cluster_tree(surf.coords, w["cfg"].leaf_size)
    bt, bs, adm = leaf_block_list(tree, w["cfg"].eta)
    log(f"[twin] {name}: surface + tree + blocks on the host ({time.perf_counter() - t0:.1f}s)")
    k_row, k_col = fx["k_row"], fx["k_col"]
    nc = len(tree.clusters)
    if k_row.shape != (nc,) or int(fx["n"]) != surf.n or int(fx["n_admissible"]) != int(adm.sum()):
        raise RuntimeError(f"{rank_fixture_path(name)} does not match the {name} structure")
    rng = np.random.default_rng(seed)
    size = np.array([c.end - c.start for c in tree.clusters])
    op = H2Matrix(tree=tree, n=surf.n)
    for c in tree.clusters:
        if c.is_leaf:
            op.row_basis[c.cid] = rng.standard_normal((c.size, int(k_row[c.cid])))
            op.col_basis[c.cid] = rng.standard_normal((c.size, int(k_col[c.cid])))
        else:
            for ch in c.children:
                op.row_transfer[ch.cid] = rng.standard_normal((int(k_row[ch.cid]), int(k_row[c.cid])))
                op.col_transfer[ch.cid] = rng.standard_normal((int(k_col[ch.cid]), int(k_col[c.cid])))
    for t, s, a in zip(bt.tolist(), bs.tolist(), adm.tolist()):
        if a:
            op.coupling.append((t, s, rng.standard_normal((int(k_row[t]), int(k_col[s])))))
        else:
            op.near.append((t, s, rng.standard_normal((int(size[t]), int(size[s])))))
    sb = op.storage_bytes()
    if sb != int(fx["storage_bytes"]):
        raise RuntimeError(f"twin storage {sb} != fixture {int(fx['storage_bytes'])}")
    log(f"[twin] {name}: {sb / 1e9:.2f} GB of seeded entries ({time.perf_counter() - t0:.1f}s)")
    return op, {"storage_bytes": sb, "n": surf.n, "build_seconds": time.perf_counter() - t0}
