"""The open-boundary potential split end to end (pipeline.py:46-63), with
both FEM solves and the H² boundary product on the GPU.

``compute_demag(mesh, m_nodal, operator)``: u1 from the deflated Neumann
solve, u2 on the boundary = M u1|boundary (the hot path: ``operator.apply``,
an ``H2Matrix`` product through libh2b for the "h2" backend), u2 inside from
the Dirichlet solve, then H = -grad(u1 + u2) and the energy.  Same inputs,
outputs and errors as the reference's ``compute_demag``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import fem

__all__ = ["PipelineResult", "compute_demag"]


@dataclass
class PipelineResult:  # pipeline.py:30-38
    u1: np.ndarray
    u2: np.ndarray
    u: np.ndarray
    h_field: np.ndarray
    e_d: float
    e_d_over_kd: float
    u1_iterations: int
    u2_iterations: int


def compute_demag(mesh, m_nodal: np.ndarray, operator, tol: float = 1e-10) -> PipelineResult:
    """pipeline.py:46-63.  ``operator`` has ``apply(u1_boundary)`` (the
    reference's ``BoundaryOperator`` or ``paper_1811_05731_b200.bem``'s)."""
    stiffness = fem.assemble_stiffness(mesh)
    u1, rep1 = fem.solve_u1(mesh, m_nodal, tol=tol, stiffness=stiffness)
    u2_boundary = operator.apply(u1[mesh.boundary_nodes])
    u2, rep2 = fem.solve_u2(mesh, u2_boundary, tol=tol, stiffness=stiffness)
    u = u1 + u2
    h = fem.compute_field(mesh, u)
    e_d, e_ratio = fem.magnetostatic_energy(mesh, m_nodal, h)
    return PipelineResult(u1=u1, u2=u2, u=u, h_field=h, e_d=e_d, e_d_over_kd=e_ratio,
                          u1_iterations=rep1.iterations, u2_iterations=rep2.iterations)
