"""The level-wise recompression (assembly/gpu_recompress.py, hmatrix/h2.py:86-183
restated with projected factors).

CPU: the algorithm, run through the numpy restatement of its kernels
(oracle/rc_ops_ref.py), against the host recompression (recompress.py, the
threaded restatement whose SVD path reproduces the reference bit for bit).
GPU (``-m gpu``): every CUDA kernel against the numpy restatement, and the
whole recompression on the device.
"""

import numpy as np
import pytest

from conftest import rel
from oracle.h2_matvec_ref import h2_matvec_ref
from oracle.rc_ops_ref import NumpyOps
from paper_1811_05731_b200.assembly import gpu_recompress as gr
from paper_1811_05731_b200.assembly.hbuild import build_cluster_tree, leaf_block_list
from paper_1811_05731_b200.assembly.recompress import recompress


def _blocks(seed, n=900, leaf=24, eta=2.0, rank=7, fallback_every=9):
    """Admissible blocks of a 1/|x-y| kernel on a random surface cloud, as
    truncated SVD factors in the batched HCA's form (B orthonormal, A's
    columns orthogonal) -- every ``fallback_every``-th block in a general form
    with full weight matrices, like the ACA fallback's."""
    rng = np.random.default_rng(seed)
    pts = rng.standard_normal((n, 3))
    pts /= np.linalg.norm(pts, axis=1)[:, None]
    pts[:, 2] *= 0.4
    tree = build_cluster_tree(pts, leaf)
    x = pts[tree.perm]
    bt, bs, adm = leaf_block_list(tree, eta)
    cl = tree.clusters
    lowrank, weights, dense = [], [], []
    for i, (t, s, a) in enumerate(zip(bt, bs, adm)):
        ct, cs = cl[int(t)], cl[int(s)]
        xt, xs = x[ct.start:ct.end], x[cs.start:cs.end]
        if not a:
            d = np.linalg.norm(xt[:, None, :] - xs[None, :, :], axis=2)
            dense.append((int(t), int(s), 1.0 / np.maximum(d, 0.05)))
            continue
        m = 1.0 / np.linalg.norm(xt[:, None, :] - xs[None, :, :], axis=2)
        u, sv, vt = np.linalg.svd(m, full_matrices=False)
        r = min(rank, int(np.sum(sv > 1e-7 * sv[0])))
        if len(lowrank) % 11 == 5:
            r = 0
        A, B = u[:, :r] * sv[:r], vt[:r].T.copy()
        if r and len(lowrank) % fallback_every == 3:
            mix = rng.standard_normal((r, r)) + 2 * np.eye(r)
            A, B = A @ mix, B @ np.linalg.inv(mix).T
            weights.append((np.linalg.qr(B)[1], np.linalg.qr(A)[1]))
        else:
            weights.append((None, np.linalg.norm(A, axis=0)))
        lowrank.append((int(t), int(s), np.ascontiguousarray(A), np.ascontiguousarray(B)))
    return tree, n, lowrank, dense, weights


@pytest.mark.parametrize("seed,leaf,eps", [(1, 24, 2e-4), (2, 16, 1e-6), (3, 40, 1e-3)])
def test_level_algorithm_matches_host_recompression(seed, leaf, eps):
    tree, n, lowrank, dense, weights = _blocks(seed, leaf=leaf)
    ref = recompress(tree, n, lowrank, dense, eps, workers=1, weights=weights)
    op = gr.recompress_gpu(tree, n, lowrank, dense, eps, weights, ops=NumpyOps())
    # the same ranks (nothing sits at the threshold in these operators) ...
    for c in tree.clusters:
        if c.is_leaf:
            assert op.row_basis[c.cid].shape == ref.row_basis[c.cid].shape
            assert op.col_basis[c.cid].shape == ref.col_basis[c.cid].shape
    assert op.storage_bytes() == ref.storage_bytes()
    assert [b[:2] for b in op.coupling] == [b[:2] for b in ref.coupling]
    # ... orthonormal nested bases ...
    for c in tree.clusters:
        if c.is_leaf:
            v = op.row_basis[c.cid]
            assert np.allclose(v.T @ v, np.eye(v.shape[1]), atol=1e-12)
        elif c.children:
            e = np.vstack([op.col_transfer[ch.cid] for ch in c.children])
            assert np.allclose(e.T @ e, np.eye(e.shape[1]), atol=1e-12)
    # ... and the same operator (bases agree up to signs, the product does not care)
    rng = np.random.default_rng(7)
    for _ in range(3):
        xv = rng.standard_normal(n)
        assert rel(h2_matvec_ref(op, xv), h2_matvec_ref(ref, xv)) < 1e-10


def test_packing_in_batches_and_oversized_blocks(monkeypatch):
    """The factor upload goes through a staging buffer in batches of whole
    clusters; a cluster's packed block larger than the buffer goes on its
    own.  Same operator as with one batch."""
    tree, n, lowrank, dense, weights = _blocks(1, n=600, leaf=24)
    want = gr.recompress_gpu(tree, n, lowrank, dense, 2e-4, weights, ops=NumpyOps())
    monkeypatch.setenv("H2B_RC_STAGE_DOUBLES", "2000")   # the largest packed block has 2590 doubles
    got = gr.recompress_gpu(tree, n, lowrank, dense, 2e-4, weights, ops=NumpyOps())
    assert all(np.array_equal(a[2], b[2]) for a, b in zip(got.coupling, want.coupling))
    assert all(np.array_equal(got.row_basis[c], want.row_basis[c]) for c in want.row_basis)
    assert all(np.array_equal(got.col_transfer[c], want.col_transfer[c]) for c in want.col_transfer)


def test_no_admissible_blocks_and_rank_zero_blocks():
    """Edge cases: an operator without admissible blocks, and one whose
    admissible blocks all have rank 0 -- every basis is empty and the product
    is the near field's, as with the host recompression."""
    tree, n, lowrank, dense, _ = _blocks(1, n=300, leaf=24)
    x = np.random.default_rng(0).standard_normal(n)
    for lr, w in (([], []),
                  ([(t, s, a[:, :0], b[:, :0]) for t, s, a, b in lowrank],
                   [(np.zeros((0, 0)), np.zeros((0, 0)))] * len(lowrank))):
        op = gr.recompress_gpu(tree, n, lr, dense, 2e-4, w, ops=NumpyOps())
        ref = recompress(tree, n, lr, dense, 2e-4, workers=1, weights=w)
        assert op.storage_bytes() == ref.storage_bytes() and len(op.coupling) == len(ref.coupling)
        assert np.array_equal(h2_matvec_ref(op, x), h2_matvec_ref(ref, x))


def test_normalise_block_keeps_the_product():
    rng = np.random.default_rng(0)
    a, b = rng.standard_normal((30, 5)), rng.standard_normal((20, 5))
    a2, b2 = gr.normalise_block(a, b)
    assert np.allclose(a2 @ b2.T, a @ b.T, atol=1e-12)
    assert np.allclose(b2.T @ b2, np.eye(5), atol=1e-12)
    g = a2.T @ a2
    assert np.allclose(g, np.diag(np.diag(g)), atol=1e-10)


def test_cuda_ops_fail_loudly_without_a_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError):
        gr.CudaOps()


# ---------------------------------------------------------------------------
# GPU: the kernels against the numpy restatement
# ---------------------------------------------------------------------------

class _Recorder(NumpyOps):
    """NumpyOps that also runs every kernel call on the GPU with the same
    inputs and compares the outputs."""

    def __init__(self):
        self.cu = gr.CudaOps()
        self.worst = {}

    def _dev(self, a):
        import torch
        return torch.from_numpy(np.ascontiguousarray(a)).cuda() if isinstance(a, np.ndarray) else a

    def _cmp(self, name, got, want, tol):
        got = got.cpu().numpy()
        scale = max(1.0, float(np.abs(want).max()))
        err = float(np.abs(got - want).max()) / scale
        self.worst[name] = max(self.worst.get(name, 0.0), err)
        assert err < tol, (name, err)

    def _both(self, name, out_idx, tol, args, post=None):
        dev = [self._dev(a) for a in args]
        getattr(NumpyOps, name)(self, *args)
        getattr(self.cu, name)(*dev)
        self.cu.sync()
        for i in out_idx:
            if post:
                post(dev[i], args[i])
            else:
                self._cmp(name, dev[i], args[i], tol)

    def leaf_gram(self, *a):
        self._both("leaf_gram", [11], 1e-13, list(a))

    def leaf_project(self, *a):
        self._both("leaf_project", [14], 1e-12, list(a))

    def inner_gram(self, *a):
        self._both("inner_gram", [6], 1e-13, list(a))

    def inner_project(self, *a):
        self._both("inner_project", [8], 1e-12, list(a))

    def extract_own(self, *a):
        self._both("extract_own", [9], 1e-13, list(a))

    def coupling(self, *a):
        self._both("coupling", [12], 1e-13, list(a))

    def eigh(self, nmat, nvec, G, ldg, lam, sweeps):
        # the Jacobi solver against LAPACK: eigenvalues, orthonormality and
        # residual (vectors of close eigenvalues may rotate among themselves)
        import torch
        g0 = G.copy()
        dG, dl = torch.from_numpy(G.copy()).cuda(), torch.from_numpy(lam.copy()).cuda()
        NumpyOps.eigh(self, nmat, nvec, G, ldg, lam, sweeps)
        self.cu.eigh(nmat, torch.from_numpy(np.ascontiguousarray(nvec)).cuda(), dG, ldg, dl, sweeps)
        self.cu.sync()
        gv, gl = dG.cpu().numpy(), dl.cpu().numpy()
        for i in range(int(nmat)):
            n = int(nvec[i])
            if n == 0:
                continue
            a = g0[i * ldg * ldg:(i + 1) * ldg * ldg].reshape(ldg, ldg)[:n, :n]
            v = gv[i * ldg * ldg:(i + 1) * ldg * ldg].reshape(ldg, ldg)[:n, :n]
            w = gl[i * ldg:i * ldg + n]
            scale = max(abs(lam[i * ldg]), 1e-300)
            assert np.all(np.diff(w) <= 1e-14 * scale)
            assert np.abs(w - lam[i * ldg:i * ldg + n]).max() <= 1e-13 * scale
            assert np.abs(v.T @ v - np.eye(n)).max() < 1e-13
            assert np.abs(a @ v - v * w[None, :]).max() <= 1e-13 * scale
        # continue with the GPU's vectors, so the later kernels see what the
        # device path sees
        G[:] = gv
        lam[:] = gl


@pytest.mark.gpu
def test_kernels_match_numpy_restatement():
    tree, n, lowrank, dense, weights = _blocks(4, n=1500, leaf=32)
    rec = _Recorder()
    op = gr.recompress_gpu(tree, n, lowrank, dense, 2e-4, weights, ops=rec)
    ref = recompress(tree, n, lowrank, dense, 2e-4, workers=1, weights=weights)
    assert set(rec.worst) == {"leaf_gram", "leaf_project", "inner_gram", "inner_project", "extract_own", "coupling"}
    xv = np.random.default_rng(1).standard_normal(n)
    assert rel(h2_matvec_ref(op, xv), h2_matvec_ref(ref, xv)) < 1e-10


@pytest.mark.gpu
@pytest.mark.parametrize("seed,leaf,eps", [(5, 64, 2e-4), (6, 24, 1e-6)])
def test_recompression_on_the_device(seed, leaf, eps):
    tree, n, lowrank, dense, weights = _blocks(seed, n=3000, leaf=leaf, rank=9)
    ref = recompress(tree, n, lowrank, dense, eps, workers=4, weights=weights)
    t = {}
    op = gr.recompress_gpu(tree, n, lowrank, dense, eps, weights, timings=t)
    assert abs(op.storage_bytes() - ref.storage_bytes()) <= 0.002 * ref.storage_bytes()
    rng = np.random.default_rng(2)
    for _ in range(2):
        xv = rng.standard_normal(n)
        assert rel(h2_matvec_ref(op, xv), h2_matvec_ref(ref, xv)) < 1e-9
    # twice the same bits
    op2 = gr.recompress_gpu(tree, n, lowrank, dense, eps, weights)
    assert all(np.array_equal(a[2], b[2]) for a, b in zip(op.coupling, op2.coupling))
    # and through the product kernel
    from paper_1811_05731_b200.h2 import h2_matvec
    xv = rng.standard_normal(n)
    assert rel(h2_matvec(op, xv), h2_matvec_ref(ref, xv)) < 1e-9
