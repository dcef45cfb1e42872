"""The oracle is pinned to the reference's own outputs (golden fixtures made
by tests/golden/make_golden.py, which runs /root/reference)."""

import numpy as np
import pytest

from conftest import load_golden, rel
from oracle.h2_matvec_ref import far_only, h2_matvec_ref, near_only


def test_oracle_matches_reference_outputs(golden):
    name, op, ex = golden
    X = ex["X"]
    for i in range(X.shape[1]):
        # same operation order as the reference: bit-identical
        assert np.array_equal(h2_matvec_ref(op, X[:, i]), ex["y_full"][:, i]), name
        assert np.array_equal(near_only(op, X[:, i]), ex["y_near"][:, i]), name
        assert np.array_equal(far_only(op, X[:, i]), ex["y_far"][:, i]), name


def test_storage_bytes_matches_reference(golden):
    name, op, ex = golden
    assert op.storage_bytes() == int(ex["storage_bytes"])


def test_h2_close_to_dense(golden):
    # reference acceptance bound: 10 * eps vs the dense oracle (test_acceptance.py:80-100)
    name, op, ex = golden
    eps = float(ex["config"][3])
    for i in range(3):
        assert rel(ex["y_full"][:, i], ex["y_dense"][:, i]) <= 10 * eps


def test_oracle_shape_error():
    op, _ = load_golden("sphere2_default")
    with pytest.raises(ValueError, match=r"vector must have shape \(162,\)"):
        h2_matvec_ref(op, np.zeros(3))


def test_sphere_mesh_restatement_is_the_reference_mesh():
    from oracle.mesh_ref import generate_sphere_mesh, mesh_hash
    _, ex = load_golden("config1_sphere4")
    mesh = generate_sphere_mesh(1.0, 4)
    assert mesh_hash(mesh) == bytes(ex["mesh_sha256"]).decode()
    assert np.array_equal(mesh.nodes[mesh.boundary_nodes], ex["boundary_coords"])


def test_energy_restatement_reproduces_reference_energy():
    from oracle.fem_ref import compute_demag
    from oracle.mesh_ref import generate_sphere_mesh
    op, ex = load_golden("config1_sphere4")
    mesh = generate_sphere_mesh(1.0, 4)
    m = np.zeros((mesh.n_nodes, 3))
    m[:, 2] = 1.0
    res = compute_demag(mesh, m, lambda u: h2_matvec_ref(op, u))
    assert res.e_d_over_kd == float(ex["energy_e_d_over_kd"])  # 0.3329597004200991
    assert abs(res.e_d_over_kd - 1 / 3) < 1e-3
    assert [res.u1_iterations, res.u2_iterations] == list(ex["energy_iterations"])
