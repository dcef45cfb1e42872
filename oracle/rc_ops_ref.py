"""TEST INFRASTRUCTURE: numpy restatement of the recompression kernels
(csrc/recompress.cu, C ABI h2b_rc_*), one Python loop per cluster, with the
kernels' data layout.  It lets the level-wise algorithm of
``paper_1811_05731_b200/assembly/gpu_recompress.py`` (hmatrix/h2.py:86-183
restated with projected factors) run on the CPU in the tests and is the
checker of the CUDA kernels in the ``-m gpu`` tests.  Never imported by the
product.
"""

from __future__ import annotations

import numpy as np


class NumpyOps:
    # -- memory: "device" arrays are numpy arrays
    def empty(self, n, dtype=np.float64):
        return np.zeros(int(max(1, n)), dtype)

    zeros = empty

    def to_device(self, a):
        return np.ascontiguousarray(a).copy() if a.size else np.zeros(1, a.dtype)

    def to_host(self, a, n=None):
        return np.array(a if n is None else a[:int(n)])

    def upload_into(self, dst, off, src):
        dst[off:off + src.size] = src

    def staging(self, n):
        return np.empty(int(n))

    def sync(self):
        pass

    # -- kernels
    @staticmethod
    def _chain_rows(c, start, end, anc, depth, foff, cown, woff, nanc, fac, wts):
        """The leaf's rows of every ancestor's own block, weighted: n x ccur."""
        n = int(end[c] - start[c])
        parts = []
        for j in range(int(depth[c]) + 1):
            a = int(anc[c * nanc + j])
            ca = int(cown[a])
            if ca == 0:
                continue
            r0 = int(start[c] - start[a])
            blk = fac[foff[a] + r0 * ca: foff[a] + (r0 + n) * ca].reshape(n, ca)
            parts.append(blk * wts[woff[a]: woff[a] + ca][None, :])
        return np.hstack(parts) if parts else np.zeros((n, 0))

    def leaf_gram(self, ids, start, end, anc, depth, foff, cown, woff, nanc, fac, wts, G, ldg):
        for i, c in enumerate(ids):
            z = self._chain_rows(int(c), start, end, anc, depth, foff, cown, woff, nanc, fac, wts)
            n = z.shape[0]
            g = G[i * ldg * ldg:(i + 1) * ldg * ldg].reshape(ldg, ldg)
            g[:n, :n] = z @ z.T

    def eigh(self, nmat, nvec, G, ldg, lam, sweeps):
        for i in range(int(nmat)):
            n = int(nvec[i])
            if n == 0:
                continue
            g = G[i * ldg * ldg:(i + 1) * ldg * ldg].reshape(ldg, ldg)
            w, v = np.linalg.eigh(g[:n, :n])
            g[:n, :n] = v[:, ::-1]
            lam[i * ldg: i * ldg + n] = w[::-1]

    def leaf_project(self, ids, start, end, anc, depth, foff, cown, woff, nanc, fac, wts, V, ldg, k, P, poff, ccur):
        for i, c in enumerate(ids):
            c = int(c)
            z = self._chain_rows(c, start, end, anc, depth, foff, cown, woff, nanc, fac, wts)
            n, kc = z.shape[0], int(k[c])
            v = V[i * ldg * ldg:(i + 1) * ldg * ldg].reshape(ldg, ldg)[:n, :kc]
            p = v.T @ z  # kc x ccur
            P[poff[c]: poff[c] + kc * z.shape[1]] = p.T.ravel()  # column-major

    @staticmethod
    def _stack(c, child, k, ccur, Pc, poffc):
        cc = int(ccur[c])
        zs = []
        for j in range(2):
            ch = int(child[2 * c + j])
            kc = int(k[ch])
            zs.append(Pc[poffc[ch]: poffc[ch] + kc * cc].reshape(cc, kc).T)
        return np.vstack(zs)  # (k1 + k2) x ccur[c]

    def inner_gram(self, ids, child, k, ccur, Pc, poffc, G, ldg):
        for i, c in enumerate(ids):
            z = self._stack(int(c), child, k, ccur, Pc, poffc)
            m = z.shape[0]
            g = G[i * ldg * ldg:(i + 1) * ldg * ldg].reshape(ldg, ldg)
            g[:m, :m] = z @ z.T

    def inner_project(self, ids, child, k, ccur, Pc, poffc, V, ldg, P, poff):
        for i, c in enumerate(ids):
            c = int(c)
            z = self._stack(c, child, k, ccur, Pc, poffc)
            m, kc = z.shape[0], int(k[c])
            v = V[i * ldg * ldg:(i + 1) * ldg * ldg].reshape(ldg, ldg)[:m, :kc]
            P[poff[c]: poff[c] + kc * z.shape[1]] = (v.T @ z).T.ravel()

    def extract_own(self, ids, parent, k, ccur, cown, woff, wts, P, poff, Q, qoff):
        for c in ids:
            c = int(c)
            kc, co = int(k[c]), int(cown[c])
            c0 = int(ccur[c]) - co
            p = P[poff[c] + kc * c0: poff[c] + kc * (c0 + co)].reshape(co, kc)
            w = wts[woff[c]: woff[c] + co]
            inv = np.where(w != 0.0, 1.0 / np.where(w != 0.0, w, 1.0), 0.0)
            Q[qoff[c]: qoff[c] + kc * co] = (p * inv[:, None]).ravel()

    def coupling(self, nb, bt, bs, rcol, ccol, kb, Qr, qoffr, kr, Qc, qoffc, kc, S, soff):
        for b in range(int(nb)):
            t, s, r = int(bt[b]), int(bs[b]), int(kb[b])
            k1, k2 = int(kr[t]), int(kc[s])
            if k1 == 0 or k2 == 0:
                continue
            qr = Qr[qoffr[t] + k1 * rcol[b]: qoffr[t] + k1 * (rcol[b] + r)].reshape(r, k1)
            qc = Qc[qoffc[s] + k2 * ccol[b]: qoffc[s] + k2 * (ccol[b] + r)].reshape(r, k2)
            S[soff[b]: soff[b] + k1 * k2] = (qr.T @ qc).ravel()
