"""GPU drop-in for the reference's Krylov solve, the step either side of
the boundary operator.

``cg_solve(a, b, tol, max_iter, deflate_constants, precond)`` replaces
``strayfield.solver.cg_solve`` (solver.py:44-98) as the reference's FEM
calls it (fem.py:79-121: ``solve_u1`` with the constant mode deflated,
``solve_u2`` on the interior block, both with
``precond=jacobi_preconditioner(a)``): the Jacobi-preconditioned CG runs as
one cooperative CUDA kernel (``csrc/cg.cu``, ``h2b_cg_*`` in
include/h2b.h).  The assembly, the field and the energy stay the
reference's own code: ``install_into_reference`` routes the reference's
``fem``/``solver`` modules to this solve (as ``h2.install_into_reference``
does for the H² product), so ``strayfield.pipeline.compute_demag`` runs with
both GPU drop-ins.  There is no CPU fallback: the solve fails loudly without
the library, and a preconditioner other than Jacobi raises
``NotImplementedError``.
"""

from __future__ import annotations

import ctypes as C
import sys
from dataclasses import dataclass

import numpy as np
from scipy.sparse import csr_matrix

from . import _native as nat

__all__ = ["SolveReport", "ConvergenceError", "GpuCG", "cg_solve", "install_into_reference"]


class ConvergenceError(RuntimeError):
    """Iterative solver failed (errors.py ConvergenceError)."""


@dataclass(frozen=True)
class SolveReport:  # solver.py:20-24
    iterations: int
    residual: float
    converged: bool


class GpuCG:
    """A sparse symmetric matrix resident on the GPU with its Jacobi
    preconditioner (``h2b_cg``); ``solve`` runs cg_solve (solver.py:44-98)."""

    def __init__(self, a):
        a = csr_matrix(a)
        a.sort_indices()
        self.n = int(a.shape[0])
        if a.shape != (self.n, self.n):
            raise ValueError("matrix must be square")
        self._rp = np.ascontiguousarray(a.indptr, np.int64)
        self._ci = np.ascontiguousarray(a.indices, np.int32)
        self._va = np.ascontiguousarray(a.data, np.float64)
        lib = nat.lib()
        h = C.c_void_p()
        rc = lib.h2b_cg_create(self.n, self._rp.ctypes.data_as(C.POINTER(C.c_int64)),
                               self._ci.ctypes.data_as(C.POINTER(C.c_int32)),
                               self._va.ctypes.data_as(C.POINTER(C.c_double)), C.byref(h))
        if rc == nat.H2B_EINVAL:
            raise ValueError(lib.h2b_last_error().decode())
        nat.check(rc, "h2b_cg_create")
        self._h = h
        self._lib = lib

    def solve(self, b, tol: float = 1e-10, max_iter: int | None = None, deflate_constants: bool = False):
        n = self.n
        if max_iter is None:
            max_iter = 10 * n
        b = np.ascontiguousarray(b, dtype=np.float64)
        if b.shape != (n,):
            raise ValueError(f"rhs must have shape ({n},)")
        b_norm = np.linalg.norm(b)
        if b_norm == 0.0:
            return np.zeros(n), SolveReport(0, 0.0, True)
        if deflate_constants and abs(b.sum()) > 1e-10 * np.abs(b).sum():  # solver.py:68-70
            raise ValueError("incompatible rhs: not orthogonal to the constant kernel")
        if max_iter <= 0:
            # solver.py:80-90: the loop never runs; x = 0, r = (deflated) b
            r = b - b.mean() if deflate_constants else b
            res = float(np.linalg.norm(r) / b_norm)
            return np.zeros(n), SolveReport(0, res, res <= tol)
        x = np.empty(n)
        it = C.c_int64(0)
        res = C.c_double(0.0)
        rc = self._lib.h2b_cg_solve(self._h, nat.as_d_ptr(b), nat.as_d_ptr(x), float(tol),
                                    int(bool(deflate_constants)), int(max_iter), C.byref(it), C.byref(res))
        if rc == nat.H2B_ECONV:
            raise ConvergenceError(self._lib.h2b_last_error().decode())
        nat.check(rc, "h2b_cg_solve")
        return x, SolveReport(int(it.value), float(res.value), float(res.value) <= tol)

    def solve_dev(self, b, tol: float = 1e-10, max_iter: int | None = None, deflate_constants: bool = False):
        """The same solve with the right-hand side and the solution in device
        memory (torch float64 CUDA tensors; ``h2b_cg_solve_dev`` on the
        current stream): what ``pipeline.compute_demag`` chains with the H²
        product without leaving the GPU.  The caller checks the deflated
        right-hand side's compatibility (solver.py:68-70)."""
        import torch
        n = self.n
        if b.shape != (n,) or b.dtype != torch.float64 or not b.is_cuda:
            raise ValueError(f"rhs must be a float64 CUDA tensor of shape ({n},)")
        if max_iter is None:
            max_iter = 10 * n
        b = b.contiguous()
        x = torch.zeros_like(b)
        b_norm = float(torch.linalg.vector_norm(b))
        if b_norm == 0.0:
            return x, SolveReport(0, 0.0, True)
        if max_iter <= 0:
            r = b - b.mean() if deflate_constants else b
            res = float(torch.linalg.vector_norm(r)) / b_norm
            return x, SolveReport(0, res, res <= tol)
        it = C.c_int64(0)
        res = C.c_double(0.0)
        rc = self._lib.h2b_cg_solve_dev(self._h, b.data_ptr(), x.data_ptr(), float(tol), int(bool(deflate_constants)),
                                        int(max_iter), C.byref(it), C.byref(res),
                                        torch.cuda.current_stream().cuda_stream)
        if rc == nat.H2B_ECONV:
            raise ConvergenceError(self._lib.h2b_last_error().decode())
        nat.check(rc, "h2b_cg_solve_dev")
        return x, SolveReport(int(it.value), float(res.value), float(res.value) <= tol)

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.h2b_cg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _is_jacobi(a, precond) -> bool:
    """Whether ``precond`` acts as diag(a)^-1 (solver.jacobi_preconditioner)."""
    d = np.asarray(a.diagonal(), dtype=np.float64)
    probe = np.random.default_rng(0).standard_normal(d.shape[0])
    with np.errstate(divide="ignore", invalid="ignore"):
        want = (1.0 / d) * probe      # solver.py:27-37: inv = 1.0 / diag; inv * r
    got = np.asarray(precond(probe), dtype=np.float64)
    return got.shape == want.shape and np.array_equal(got, want)


def cg_solve(a, b, tol: float = 1e-10, max_iter: int | None = None, deflate_constants: bool = False,
             precond="jacobi"):
    """solver.py:44-98 with the Jacobi preconditioner, on the GPU.  Same
    signature as the reference; ``precond`` must be the reference's
    ``jacobi_preconditioner(a)`` (what fem.py passes) or "jacobi"."""
    if not (isinstance(precond, str) and precond == "jacobi") and not (callable(precond) and _is_jacobi(a, precond)):
        raise NotImplementedError("the GPU solve is Jacobi-preconditioned CG "
                                  "(precond=jacobi_preconditioner(a), as fem.py:91-93, 118-119 pass it)")
    solver = GpuCG(a)
    try:
        return solver.solve(b, tol=tol, max_iter=max_iter, deflate_constants=deflate_constants)
    finally:
        solver.close()


def install_into_reference(solver_module, fem_module=None) -> None:
    """Route the reference's solves to the GPU: ``strayfield.solver.cg_solve``
    and the name ``strayfield.fem`` imported from it (fem.py:15, called at
    fem.py:91, 118).  Its SolveReport and ConvergenceError types are the
    ones returned and raised."""
    ref_report = getattr(solver_module, "SolveReport", SolveReport)
    ref_error = getattr(sys.modules.get(solver_module.__name__.rsplit(".", 1)[0] + ".errors"),
                        "ConvergenceError", ConvergenceError)

    def ref_cg_solve(a, b, tol=1e-10, max_iter=None, deflate_constants=False, precond=None):
        if precond is None:
            raise NotImplementedError("the GPU solve is Jacobi-preconditioned CG")
        try:
            x, rep = cg_solve(a, b, tol=tol, max_iter=max_iter, deflate_constants=deflate_constants,
                              precond=precond)
        except ConvergenceError as e:
            raise ref_error(str(e)) from None
        return x, ref_report(rep.iterations, rep.residual, rep.converged)

    ref_cg_solve.__doc__ = cg_solve.__doc__
    solver_module.cg_solve = ref_cg_solve
    if fem_module is not None:
        fem_module.cg_solve = ref_cg_solve
