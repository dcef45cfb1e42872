"""GPU Jacobi-PCG (csrc/cg.cu) on a structured tetrahedral cube mesh: time per
solve and per iteration, HBM bytes per iteration, and the oracle's CPU CG
(solver.py:44-98 restated) on the same system.

    python tools/cg_bench.py [--n 64] [--cpu]

The mesh is [0,1]^3 cut into n^3 cubes of 6 tetrahedra (Kuhn split); the
system is the deflated Neumann problem of solve_u1 (fem.py:79-95) with a
seeded random magnetization.  Bytes per iteration (algorithmic): the CSR
matrix (8 + 4 bytes per entry + 8 per row) read once, p gathered once per
entry's row (counted once: n doubles), and the vector updates (x, r, z, p,
ap, inv: 9 n doubles read or written)."""

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


class CubeMesh:
    def __init__(self, n):
        g = np.arange(n + 1)
        x, y, z = np.meshgrid(g, g, g, indexing="ij")
        self.nodes = np.stack([x.ravel(), y.ravel(), z.ravel()], axis=1) / n
        idx = lambda i, j, k: (i * (n + 1) + j) * (n + 1) + k
        i, j, k = [a.ravel() for a in np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")]
        c = [idx(i + (b >> 2 & 1), j + (b >> 1 & 1), k + (b & 1)) for b in range(8)]
        # Kuhn split of the cube along the main diagonal c0 -> c7
        paths = [(0, 1, 3, 7), (0, 1, 5, 7), (0, 2, 3, 7), (0, 2, 6, 7), (0, 4, 5, 7), (0, 4, 6, 7)]
        tets = np.concatenate([np.stack([c[a], c[b], c[d], c[e]], axis=1) for a, b, d, e in paths])
        p = self.nodes[tets]
        vol = np.einsum("ij,ij->i", p[:, 1] - p[:, 0], np.cross(p[:, 2] - p[:, 0], p[:, 3] - p[:, 0]))
        tets[vol < 0] = tets[vol < 0][:, [0, 2, 1, 3]]
        self.tets = tets
        self.n_nodes = self.nodes.shape[0]
        on_b = ((self.nodes == 0) | (self.nodes == 1)).any(axis=1)
        self.boundary_nodes = np.flatnonzero(on_b)
        self.n_boundary = self.boundary_nodes.size


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--cpu", action="store_true", help="also time the oracle CG on one core")
    a = ap.parse_args()
    import torch
    import __graft_entry__
    __graft_entry__.build()
    from oracle.fem_ref import rhs_u1, stiffness
    from paper_1811_05731_b200 import fem
    mesh = CubeMesh(a.n)
    A = stiffness(mesh)
    m = np.random.default_rng(3).standard_normal((mesh.n_nodes, 3))
    b = rhs_u1(mesh, m)
    solver = fem.GpuCG(A)
    x, rep = solver.solve(b, deflate_constants=True)
    ts = []
    for _ in range(a.reps):
        t = time.perf_counter()
        x, rep = solver.solve(b, deflate_constants=True)
        ts.append(time.perf_counter() - t)
    t = float(np.median(ts))
    n, nnz = mesh.n_nodes, A.nnz
    bytes_it = 12 * nnz + 8 * (n + 1) + 8 * n + 8 * 9 * n
    out = {"mesh": f"cube {a.n}^3 Kuhn tets", "n": n, "nnz": int(nnz), "iterations": rep.iterations,
           "residual": rep.residual, "solve_ms": 1e3 * t, "us_per_iteration": 1e6 * t / max(1, rep.iterations),
           "bytes_per_iteration": bytes_it, "GB/s": bytes_it * rep.iterations / t / 1e9,
           "note": "solve time includes the host<->device copies of b and x"}
    if a.cpu:
        from oracle.fem_ref import _pcg
        tc = time.perf_counter()
        xo, ito = _pcg(A, b, 1e-10, True)
        tc = time.perf_counter() - tc
        out.update(cpu_oracle_ms=1e3 * tc, cpu_oracle_iterations=ito,
                   rel_diff_vs_oracle=float(np.linalg.norm(x - xo) / np.linalg.norm(xo)))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
