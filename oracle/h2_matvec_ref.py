"""CPU restatement of the reference H² matvec — TEST INFRASTRUCTURE ONLY.

Follows /root/reference/pkg/src/strayfield/hmatrix/h2.py:186-244 step by
step (the four loops and their accumulation order), restated with explicit
post-/pre-order traversals instead of recursion.  It also serves as the
"port" CPU baseline of bench.py: like the reference it is a Python loop over
small numpy GEMVs, so it has the reference's cost profile.

Accepts any object with the H2Matrix fields (reference or mirror).
"""

from __future__ import annotations

import numpy as np

__all__ = ["h2_matvec_ref", "near_only", "far_only"]


def _postorder(root):
    out, stack = [], [(root, False)]
    while stack:
        c, seen = stack.pop()
        if seen or c.is_leaf:
            out.append(c)
            continue
        stack.append((c, True))
        for ch in reversed(c.children):
            stack.append((ch, False))
    return out


def h2_matvec_ref(op, x, *, use_far: bool = True, use_near: bool = True) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)                       # h2.py:188
    if x.shape != (op.n,):                                    # h2.py:189-190
        raise ValueError(f"vector must have shape ({op.n},)")
    tree = op.tree
    perm = tree.perm
    xp = x[perm]                                              # h2.py:192-193
    yp = np.zeros(op.n)                                       # h2.py:221
    if use_far:
        # forward transform, leaves to root (h2.py:195-209)
        x_hat = {}
        for c in _postorder(tree.root):
            if c.is_leaf:
                x_hat[c.cid] = op.col_basis[c.cid].T @ xp[c.start:c.end]
            else:
                acc = None
                for ch in c.children:
                    part = op.col_transfer[ch.cid].T @ x_hat[ch.cid]
                    acc = part if acc is None else acc + part
                x_hat[c.cid] = acc
        # coupling, in block-list order (h2.py:211-218)
        y_hat = {}
        for rcid, ccid, s_b in op.coupling:
            contrib = s_b @ x_hat[ccid]
            y_hat[rcid] = contrib if rcid not in y_hat else y_hat[rcid] + contrib
        # backward transform, root to leaves (h2.py:220-235)
        stack = [(tree.root, None)]
        while stack:
            c, coeff = stack.pop()
            own = y_hat.get(c.cid)
            if own is not None:
                coeff = own if coeff is None else coeff + own
            if c.is_leaf:
                if coeff is not None:
                    yp[c.start:c.end] += op.row_basis[c.cid] @ coeff
                continue
            for ch in reversed(c.children):
                down = None if coeff is None else op.row_transfer[ch.cid] @ coeff
                stack.append((ch, down))
    if use_near:
        clusters = tree.clusters
        for rcid, ccid, mat in op.near:                       # h2.py:237-240
            rc, cc = clusters[rcid], clusters[ccid]
            yp[rc.start:rc.end] += mat @ xp[cc.start:cc.end]
    y = np.zeros(op.n)                                        # h2.py:242-244
    y[perm] = yp
    return y


def near_only(op, x):
    """Reference product of the ablated operator with ``coupling=[]``
    (SURVEY §4): the near field alone."""
    return h2_matvec_ref(op, x, use_far=False)


def far_only(op, x):
    """Reference product of the ablated operator with ``near=[]``."""
    return h2_matvec_ref(op, x, use_near=False)
