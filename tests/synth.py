"""Random H² operators with adversarial structure, for layout/kernel tests.

Real operators built by the reference have leaves <= leaf_size, ranks well
below 64 and leaf x leaf near blocks.  These random ones also exercise the
general paths of the planner and kernel: leaves and ranks above 64 rows
(row tiles), rank-0 clusters, zero-size coupling blocks, near blocks whose
row and/or column cluster is not a leaf, repeated blocks and heavy rows.
The product semantics are the reference's (h2.py:186-244), evaluated by
oracle.h2_matvec_ref.
"""

from __future__ import annotations

import numpy as np

from paper_1811_05731_b200.cluster import Cluster, ClusterTree
from paper_1811_05731_b200.h2 import H2Matrix


def random_tree(rng, n: int, max_leaf: int) -> ClusterTree:
    clusters: list[Cluster] = []

    def rec(start, end):
        c = Cluster(start, end, np.zeros(3), np.ones(3))
        if end - start > max_leaf or (end - start >= 2 and rng.random() < 0.15 and start > 0):
            mid = int(rng.integers(start + 1, end))
            c.children = (rec(start, mid), rec(mid, end))
        return c

    root = rec(0, n)

    def number(c):
        c.cid = len(clusters)
        clusters.append(c)
        for ch in c.children:
            number(ch)

    number(root)
    return ClusterTree(root=root, perm=rng.permutation(n).astype(np.int64), clusters=clusters)


def random_h2(seed: int, n: int = 700, max_leaf: int = 90, max_rank: int = 80,
              n_coupling: int = 300, n_near: int = 200) -> H2Matrix:
    rng = np.random.default_rng(seed)
    tree = random_tree(rng, n, max_leaf)
    cl = tree.clusters
    nc = len(cl)
    k_row = rng.integers(0, max_rank + 1, nc)
    k_col = rng.integers(0, max_rank + 1, nc)
    # a few rank-0 clusters and small ranks, like the top of real trees
    k_row[rng.random(nc) < 0.15] = 0
    k_col[rng.random(nc) < 0.15] = 0
    k_row[0] = k_col[0] = 0
    op = H2Matrix(tree=tree, n=n)
    for c in cl:
        if c.is_leaf:
            op.row_basis[c.cid] = rng.standard_normal((c.size, k_row[c.cid]))
            op.col_basis[c.cid] = rng.standard_normal((c.size, k_col[c.cid]))
        for ch in c.children:
            op.row_transfer[ch.cid] = rng.standard_normal((k_row[ch.cid], k_row[c.cid]))
            op.col_transfer[ch.cid] = rng.standard_normal((k_col[ch.cid], k_col[c.cid]))
    for _ in range(n_coupling):
        t = int(rng.integers(nc))
        s = int(rng.integers(nc))
        op.coupling.append((t, s, rng.standard_normal((k_row[t], k_col[s]))))
    # one heavy coupling row
    heavy = int(rng.integers(nc))
    for _ in range(40):
        s = int(rng.integers(nc))
        op.coupling.append((heavy, s, rng.standard_normal((k_row[heavy], k_col[s]))))
    leaves = [c for c in cl if c.is_leaf]
    for i in range(n_near):
        t = leaves[int(rng.integers(len(leaves)))] if rng.random() < 0.8 else cl[int(rng.integers(nc))]
        s = leaves[int(rng.integers(len(leaves)))] if rng.random() < 0.8 else cl[int(rng.integers(nc))]
        op.near.append((t.cid, s.cid, rng.standard_normal((t.size, s.size))))
    # one heavy near row
    t = leaves[0]
    for _ in range(30):
        s = leaves[int(rng.integers(len(leaves)))]
        op.near.append((t.cid, s.cid, rng.standard_normal((t.size, s.size))))
    return op
