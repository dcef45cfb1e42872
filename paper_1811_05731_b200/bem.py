"""Backend-agnostic boundary-operator contract (u1|boundary -> u2|boundary).

Mirrors ``BoundaryOperator`` / ``apply_operator``
(/root/reference/pkg/src/strayfield/bem.py:246-284): float64 coercion, exact
shape check with the reference's message, then dispatch on the backend.  The
``"h2"`` backend's payload is an ``H2Matrix`` (mirror or reference object)
whose product runs on the GPU.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .h2 import h2_matvec

__all__ = ["BoundaryOperator", "apply_operator"]


@dataclass(frozen=True)
class BoundaryOperator:
    backend: str            # "dense" | "h2"
    n: int
    diag: np.ndarray        # Psi/4pi - 1, kept for introspection only
    payload: object

    def apply(self, u1_boundary: np.ndarray) -> np.ndarray:
        return apply_operator(self, u1_boundary)

    def storage_bytes(self) -> int:
        if self.backend == "dense":
            return self.payload.size * 8
        return self.payload.storage_bytes()


def apply_operator(op: BoundaryOperator, u1_boundary: np.ndarray) -> np.ndarray:
    u1_boundary = np.asarray(u1_boundary, dtype=np.float64)
    if u1_boundary.shape != (op.n,):
        raise ValueError(f"vector must have shape ({op.n},)")
    if op.backend == "dense":
        return op.payload @ u1_boundary
    if op.backend == "h2":
        return h2_matvec(op.payload, u1_boundary)
    raise ValueError(f"unknown backend '{op.backend}'")
