"""CPU restatement of the collocation entries — TEST INFRASTRUCTURE ONLY.

Restates /root/reference/pkg/src/strayfield/bem.py:99-153 (``_panel_rows``:
closed-form integrals of shape function x dG/dn over flat triangles) and the
row assembly of ``row_for_point`` / ``block`` (bem.py:207-235: scatter with
np.add.at over the triangles incident to the columns, then the diagonal
term).  It checks the GPU collocation kernel (csrc/colloc.cu) and stands in
for it when the operator builder is exercised by CPU-only tests.
"""

from __future__ import annotations

import math

import numpy as np

__all__ = ["panel_rows", "CpuCollocation"]

_FOUR_PI = 4.0 * math.pi


def panel_rows(x: np.ndarray, P: np.ndarray) -> np.ndarray:
    """(T, 3) values for point x and panel table rows P (T, 34)."""
    verts = P[:, 0:9].reshape(-1, 3, 3)
    nhat = P[:, 9:12]
    grads = P[:, 12:21].reshape(-1, 3, 3)
    gm = P[:, 21:30].reshape(-1, 3, 3)
    cop_scale = P[:, 30]
    slen = P[:, 31:34]
    rho = verts - x[None, None, :]
    r = np.linalg.norm(rho, axis=2)
    a, b, c = rho[:, 0], rho[:, 1], rho[:, 2]
    ra, rb, rc = r[:, 0], r[:, 1], r[:, 2]
    det = np.einsum("tj,tj->t", a, np.cross(b, c))
    den = (ra * rb * rc + np.einsum("tj,tj->t", a, b) * rc + np.einsum("tj,tj->t", b, c) * ra
           + np.einsum("tj,tj->t", c, a) * rb)
    omega = 2.0 * np.arctan2(det, den)
    zeta = np.einsum("tj,tj->t", nhat, a)
    coplanar = np.abs(zeta) <= 1e-12 * np.maximum(r.max(axis=1), cop_scale)
    proj = x[None, :] + zeta[:, None] * nhat
    lam = 1.0 + np.einsum("tid,tid->ti", grads, proj[:, None, :] - verts)
    r_pair = np.stack([ra + rb, rb + rc, rc + ra], axis=1)
    num = r_pair + slen
    dnm = r_pair - slen
    safe = dnm > 0.0
    p_edge = np.zeros_like(num)
    np.log(np.divide(num, dnm, out=np.ones_like(num), where=safe), out=p_edge, where=safe)
    vals = -(lam * omega[:, None] - zeta[:, None] * np.einsum("tie,te->ti", gm, p_edge)) / _FOUR_PI
    vals[coplanar] = 0.0
    return vals


class CpuCollocation:
    """Same call signature as the GPU evaluator of the operator builder."""

    def __init__(self, surface, panels, inc):
        self.tri = surface.triangles
        self.panels = panels
        self.inc_ptr, self.inc_tri, _ = inc
        self.diag = surface.diag
        self.n = surface.n

    def rows(self, points, col_begin, col_count, diag_node, out_off, colidx, out_len):
        out = np.zeros(out_len)
        local = np.full(self.n, -1, dtype=np.int64)
        for j in range(points.shape[0]):
            cols = colidx[col_begin[j]: col_begin[j] + col_count[j]]
            parts = [self.inc_tri[self.inc_ptr[v]: self.inc_ptr[v + 1]] for v in cols]
            sel = np.unique(np.concatenate(parts)) if parts else np.zeros(0, np.int64)
            vals = panel_rows(points[j], self.panels[sel])
            local[cols] = np.arange(cols.size)
            dest = local[self.tri[sel]]
            keep = dest >= 0
            row = np.zeros(cols.size)
            np.add.at(row, dest[keep], vals[keep])
            dn = diag_node[j]
            if dn >= 0 and local[dn] >= 0:
                row[local[dn]] += self.diag[dn]
            local[cols] = -1
            out[out_off[j]: out_off[j] + cols.size] = row
        return out
