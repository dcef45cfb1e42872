"""GPU parity: the sm_100a kernel (through the C ABI) against the reference's
own outputs and the oracle.

Tolerance (north_star): relative l2 error <= 1e-12 in fp64.  The far field
is checked on its own (ablated operator, near=[]) because it is only ~2% of
||y|| for random inputs and would be diluted in the full product.
"""

import dataclasses

import numpy as np
import pytest

from conftest import load_golden, rel
from oracle.h2_matvec_ref import h2_matvec_ref

pytestmark = pytest.mark.gpu
TOL = 1e-12


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()


def _gpu():
    from paper_1811_05731_b200 import h2
    return h2


def test_full_product_matches_reference(golden):
    name, op, ex = golden
    h2 = _gpu()
    X = ex["X"]
    for i in range(X.shape[1]):
        y = h2.h2_matvec(op, X[:, i])
        assert rel(y, ex["y_full"][:, i]) <= TOL, (name, i)


def test_far_and_near_fields_separately(golden):
    name, op, ex = golden
    h2 = _gpu()
    x = ex["X"][:, 0]
    far = dataclasses.replace(op, near=[])
    near = dataclasses.replace(op, coupling=[])
    if op.coupling:
        assert rel(h2.h2_matvec(far, x), ex["y_far"][:, 0]) <= TOL, name
    assert rel(h2.h2_matvec(near, x), ex["y_near"][:, 0]) <= TOL, name


@pytest.mark.parametrize("opts", [dict(task_bytes=512), dict(task_bytes=4096, sched_flags=1),
                                  dict(warps_per_cta=4, ctas_per_sm=1),
                                  dict(task_bytes=2048, sched_flags=(15 << 20) | (6 << 26)),
                                  dict(sched_flags=(2 << 20) | (8 << 26)),
                                  dict(sched_flags=(3 << 4) | (3 << 26)),
                                  dict(task_bytes=8192, sched_flags=(8 << 4)),
                                  dict(sched_flags=4), dict(task_bytes=1024, sched_flags=4 | (8 << 4) | (6 << 26))])
def test_plan_variants(opts):
    op, ex = load_golden("config1_sphere4")
    dev = _gpu().DeviceOperator(op, **opts)
    try:
        for i in range(3):
            assert rel(dev.matvec(ex["X"][:, i]), ex["y_full"][:, i]) <= TOL
    finally:
        dev.close()


@pytest.mark.parametrize("nrhs", [2, 4, 8, 16])
def test_multi_rhs(nrhs):
    op, ex = load_golden("config1_sphere4")
    X = np.tile(ex["X"], (1, 4))[:, :nrhs]
    Yref = np.tile(ex["y_full"], (1, 4))[:, :nrhs]
    Y = _gpu().h2_matmat(op, X)
    for i in range(nrhs):
        assert rel(Y[:, i], Yref[:, i]) <= TOL


@pytest.mark.parametrize("name", ["config1_sphere4", "prism_20_40_2_default"])
@pytest.mark.parametrize("nrhs", [8, 16])
def test_multi_rhs_ring_matches_register_path(name, nrhs):
    """The TMA-ring streaming of the DMMA items (default) groups columns into
    k-steps exactly like the register-staged loop (H2B_SCHED_NO_RING), so
    the two give bit-identical products; both match the reference."""
    op, ex = load_golden(name)
    h2 = _gpu()
    rng = np.random.default_rng(7)
    X = rng.standard_normal((op.n, nrhs))
    ys = []
    for flags in (0, h2.SCHED_NO_RING):
        dev = h2.DeviceOperator(op, sched_flags=flags)
        try:
            ys.append(dev.matvec(X))
        finally:
            dev.close()
    assert np.array_equal(ys[0], ys[1])
    for i in range(nrhs):
        assert rel(ys[0][:, i], h2_matvec_ref(op, X[:, i])) <= TOL


@pytest.mark.parametrize("name", ["config1_sphere4", "prism_20_40_2_default", "torus_32_16_4_default"])
def test_ring_warps_bit_identical(name):
    """Single-vector items streamed through a warp's TMA ring run the same
    column-ordered FMA chain as register-streamed ones: any mix of ring and
    register warps gives the same bits."""
    op, ex = load_golden(name)
    h2 = _gpu()
    x = ex["X"][:, 0]
    ys = []
    for flags in (0, h2.SCHED_RING_WARPS(3) | h2.SCHED_NEAR_PRIO(3), h2.SCHED_RING_WARPS(8)):
        dev = h2.DeviceOperator(op, sched_flags=flags)
        try:
            ys.append(dev.matvec(x))
        finally:
            dev.close()
    assert np.array_equal(ys[0], ys[1]) and np.array_equal(ys[0], ys[2])
    assert rel(ys[0], ex["y_full"][:, 0]) <= TOL


def test_effective_sched_flags_reported():
    """Small operators keep plain scheduling (the streaming defaults start
    at H2B_STREAM_DEFAULT_BYTES per rank) with leaf mix 2; explicit flags are
    used as given and reported back through h2b_stats."""
    op, ex = load_golden("config1_sphere4")
    h2 = _gpu()
    dev = h2.DeviceOperator(op)
    try:
        st = dev.stats()
        assert st["sched_flags"] == h2.SCHED_LEAF_MIX(2) and st["ring_warps"] == 0
    finally:
        dev.close()
    flags = h2.SCHED_EXPLICIT | h2.SCHED_RING_WARPS(8) | (2 << 18) | h2.SCHED_NEAR_PRIO(6) | h2.SCHED_LEAF_MIX(2)
    dev = h2.DeviceOperator(op, sched_flags=flags, far_task_bytes=8192)
    try:
        st = dev.stats()
        assert st["sched_flags"] == flags and st["ring_warps"] == 8
        assert rel(dev.matvec(ex["X"][:, 0]), ex["y_full"][:, 0]) <= TOL
    finally:
        dev.close()


STREAMING = dict(sched_flags=8 | (8 << 4) | (2 << 18) | (6 << 26) | (4 << 20) | (1 << 25), far_task_bytes=8192, task_bytes=262144)


@pytest.mark.parametrize("nrhs", [2, 4])
def test_ring_multi_bit_identical(nrhs):
    """2 and 4 right-hand sides through the TMA ring give the same bits as
    the register-streamed path."""
    op, ex = load_golden("prism_20_40_2_default")
    h2 = _gpu()
    X = np.random.default_rng(11).standard_normal((op.n, nrhs))
    ys = []
    for flags in (8 | (8 << 4) | (2 << 18), 8 | (8 << 4) | (2 << 18) | h2.SCHED_NO_RING):
        dev = h2.DeviceOperator(op, sched_flags=flags)
        try:
            ys.append(dev.matvec(X))
        finally:
            dev.close()
    assert np.array_equal(ys[0], ys[1])
    for i in range(nrhs):
        assert rel(ys[0][:, i], h2_matvec_ref(op, X[:, i])) <= TOL


@pytest.mark.parametrize("nrhs", [1, 2, 4, 8, 16])
def test_streaming_defaults_every_nrhs(nrhs):
    """The scheduling large operators get (ring warps with 4 KB stages,
    near-priority warps, leaf mix, 8 KB chain pieces staged in the ring,
    evict-first copies), forced on small ones, for every right-hand-side
    count: results within the parity bound."""
    op, ex = load_golden("prism_20_40_2_default")
    h2 = _gpu()
    rng = np.random.default_rng(nrhs)
    X = rng.standard_normal((op.n, nrhs))
    dev = h2.DeviceOperator(op, **STREAMING)
    try:
        Y = dev.matvec(X[:, 0] if nrhs == 1 else X)
    finally:
        dev.close()
    Y = Y.reshape(op.n, nrhs)
    for i in range(nrhs):
        assert rel(Y[:, i], h2_matvec_ref(op, X[:, i])) <= TOL


@pytest.mark.parametrize("seed", range(3))
def test_random_structures(seed):
    from synth import random_h2
    op = random_h2(seed)
    h2 = _gpu()
    rng = np.random.default_rng(seed)
    for _ in range(2):
        x = rng.standard_normal(op.n)
        assert rel(h2.h2_matvec(op, x), h2_matvec_ref(op, x)) <= TOL
    for nrhs in (4, 8, 16):  # CUDA-core path and the DMMA path (8, 16)
        X = rng.standard_normal((op.n, nrhs))
        Y = h2.h2_matmat(op, X)
        for i in range(nrhs):
            assert rel(Y[:, i], h2_matvec_ref(op, X[:, i])) <= TOL


def test_zero_linearity_determinism():
    op, ex = load_golden("config1_sphere4")
    h2 = _gpu()
    assert np.array_equal(h2.h2_matvec(op, np.zeros(op.n)), np.zeros(op.n))
    rng = np.random.default_rng(1234)
    x, y = rng.standard_normal((2, op.n))
    lhs = h2.h2_matvec(op, 2.0 * x + 0.5 * y)
    rhs = 2.0 * h2.h2_matvec(op, x) + 0.5 * h2.h2_matvec(op, y)
    assert np.linalg.norm(lhs - rhs) <= 1e-12 * np.linalg.norm(lhs)
    # deterministic (no float atomics): repeated products and a reloaded
    # copy of the operator are bit-identical (cf. test_hmatrix.py:349-357)
    a = h2.h2_matvec(op, x)
    for _ in range(5):
        assert np.array_equal(h2.h2_matvec(op, x), a)
    from paper_1811_05731_b200.io import h2_from_arrays, h2_to_arrays
    copy = h2_from_arrays(h2_to_arrays(op))
    assert np.array_equal(h2.h2_matvec(copy, x), a)


def test_shape_errors_and_input_untouched():
    op, ex = load_golden("sphere2_default")
    h2 = _gpu()
    with pytest.raises(ValueError, match=r"vector must have shape \(162,\)"):
        h2.h2_matvec(op, np.zeros(3))
    with pytest.raises(ValueError):
        h2.h2_matvec(op, np.zeros((162, 1)))
    x = ex["X"][:, 0].copy()
    x0 = x.copy()
    h2.h2_matvec(op, x)
    assert np.array_equal(x, x0)
    # list input is coerced like np.asarray(x, float64)
    assert rel(h2.h2_matvec(op, list(x)), ex["y_full"][:, 0]) <= TOL


def test_boundary_operator_contract():
    from paper_1811_05731_b200.bem import BoundaryOperator
    op, ex = load_golden("sphere3_l32_eta2_o4")
    bop = BoundaryOperator(backend="h2", n=op.n, diag=np.zeros(op.n), payload=op)
    assert rel(bop.apply(ex["X"][:, 1]), ex["y_full"][:, 1]) <= TOL
    assert bop.storage_bytes() == int(ex["storage_bytes"])
    with pytest.raises(ValueError, match="vector must have shape"):
        bop.apply(np.zeros(op.n + 1))


def test_stream_bytes_equals_storage_bytes(golden):
    name, op, ex = golden
    dev = _gpu().device_operator(op)
    assert dev.stream_bytes() == op.storage_bytes() == int(ex["storage_bytes"])


def test_device_pointer_path_with_torch():
    import torch
    op, ex = load_golden("config1_sphere4")
    dev = _gpu().device_operator(op)
    x = torch.from_numpy(ex["X"][:, 0]).cuda()
    y = torch.empty_like(x)
    s = torch.cuda.current_stream()
    dev.matvec_dev(x.data_ptr(), y.data_ptr(), 1, s.cuda_stream)
    s.synchronize()
    assert rel(y.cpu().numpy(), ex["y_full"][:, 0]) <= TOL


def test_sphere_energy_matches_reference():
    """Uniformly magnetized sphere: compute_demag (pipeline.py:46-63) with the
    GPU product in the middle reproduces the reference energy."""
    from oracle.fem_ref import compute_demag
    from oracle.mesh_ref import generate_sphere_mesh, mesh_hash
    op, ex = load_golden("config1_sphere4")
    mesh = generate_sphere_mesh(1.0, 4)
    assert mesh_hash(mesh) == bytes(ex["mesh_sha256"]).decode()
    m = np.zeros((mesh.n_nodes, 3))
    m[:, 2] = 1.0
    res = compute_demag(mesh, m, lambda u: _gpu().h2_matvec(op, u))
    ref = float(ex["energy_e_d_over_kd"])   # 0.3329597004200991
    assert abs(res.e_d_over_kd - ref) <= 1e-12 * abs(ref)
    assert rel(res.u2_boundary, ex["energy_u2_boundary"]) <= TOL


def test_reference_test_patterns_against_dense(golden):
    """The reference's own H²-vs-dense bounds (test_hmatrix.py:272-287,
    test_acceptance.py:80-100) hold for the GPU product."""
    name, op, ex = golden
    h2 = _gpu()
    eps = float(ex["config"][3])
    for i in range(3):
        assert rel(h2.h2_matvec(op, ex["X"][:, i]), ex["y_dense"][:, i]) <= 10 * eps


@pytest.mark.parametrize("name", ["config1_sphere4", "prism_20_40_2_default", "random"])
@pytest.mark.parametrize("nrhs", [8, 16])
def test_multi_rhs_near_split_bit_identical(name, nrhs, monkeypatch):
    """8/16 right-hand sides run the near field in a lean kernel (TMA for
    both operands, 2 or 3 stages; or the ring + register-gather variant with
    both stage sizes) and the rest in the dataflow kernel: the same per-item DMMA k-steps and the same fixed-order slot
    sums as the single dataflow launch (H2B_NEAR_SPLIT=0), so the same bits;
    all match the oracle.  "random": leaves above 64 nodes (row tiles whose
    near items take the register-staged fallback)."""
    if name == "random":
        from synth import random_h2
        op = random_h2(3)
    else:
        op, _ = load_golden(name)
    h2 = _gpu()
    X = np.random.default_rng(17).standard_normal((op.n, nrhs))
    ys = {}
    # (all on the classic plan, H2B_STAGED=0: a staged plan cuts the far-field
    # pieces differently, so its partial sums differ in the last bits)
    variants = {"fused": {"H2B_NEAR_SPLIT": "0"},
                "ring8k": {"H2B_NEAR_IMPL": "ring", "H2B_NEAR_STAGE": "8192"},
                "ring4k": {"H2B_NEAR_IMPL": "ring", "H2B_NEAR_STAGE": "4096"},
                "tma2": {}, "tma3": {"H2B_NEAR_NST": "3"}, "staged": {"H2B_MRHS_RING_ALL": "0"}}
    for name_v, env in variants.items():
        for k in ("H2B_NEAR_SPLIT", "H2B_NEAR_IMPL", "H2B_NEAR_STAGE", "H2B_NEAR_NST", "H2B_MRHS_RING_ALL", "H2B_STAGED"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        monkeypatch.setenv("H2B_STAGED", "0")
        dev = h2.DeviceOperator(op)
        try:
            ys[name_v] = dev.matvec(X)
        finally:
            dev.close()
    for name_v in variants:
        assert np.array_equal(ys["fused"], ys[name_v]), name_v
    for i in range(nrhs):
        assert rel(ys["tma2"][:, i], h2_matvec_ref(op, X[:, i])) <= TOL


@pytest.mark.parametrize("nrhs", [1, 16])
@pytest.mark.parametrize("flags", ["skip", "gate", "skip+gate", "none"])
def test_level_skipping_chain_on_gpu(golden, nrhs, flags):
    """The level-skipping far-field chain (H2B_PLAN_SKIP_LEVELS) and the gated
    coupling rows (H2B_PLAN_GATE) on the GPU, alone and together: the same
    product to rounding (1e-12), the far field checked on its own."""
    name, op, ex = golden
    h2 = _gpu()
    pf = {"skip": h2.PLAN_SKIP_LEVELS, "gate": h2.PLAN_GATE | h2.PLAN_NO_SKIP,
          "skip+gate": h2.PLAN_SKIP_LEVELS | h2.PLAN_GATE, "none": h2.PLAN_NO_SKIP | h2.PLAN_NO_GATE}[flags]
    X = np.random.default_rng(23).standard_normal((op.n, nrhs))
    for o in (op, dataclasses.replace(op, near=[])):
        dev = h2.DeviceOperator(o, plan_flags=pf)
        try:
            Y = dev.matvec(X[:, 0] if nrhs == 1 else X).reshape(op.n, nrhs)
            Y2 = dev.matvec(X[:, 0] if nrhs == 1 else X).reshape(op.n, nrhs)
        finally:
            dev.close()
        assert np.array_equal(Y, Y2)
        for i in range(nrhs):
            ref = h2_matvec_ref(o, X[:, i])
            if np.linalg.norm(ref) > 0:
                assert rel(Y[:, i], ref) <= TOL, (name, i)


@pytest.mark.gpu
def test_operator_beyond_l2_and_staged_host_copies(monkeypatch):
    """h2b_matvec can stage vectors of >= 1 MB through pinned memory with
    copy threads (H2B_COPY_THREADS; pageable numpy arrays are what
    apply_operator / compute_demag pass).  A block-diagonal operator with
    327 680 nodes and 168 MB of near-field blocks -- larger than the 126 MB
    L2, so every product streams from HBM, unlike the golden operators: the
    plain path (default), the staged path with 2 and 7 threads and numpy
    agree; 1 and 2 right-hand sides, repeated calls."""
    from paper_1811_05731_b200.cluster import Cluster, ClusterTree
    from paper_1811_05731_b200.h2 import DeviceOperator, H2Matrix
    rng = np.random.default_rng(5)
    leaf, nleaf = 64, 5120
    n = leaf * nleaf
    clusters = []

    def build(lo, hi):
        c = Cluster(lo * leaf, hi * leaf, np.zeros(3), np.ones(3))
        c.cid = len(clusters)
        clusters.append(c)
        if hi - lo > 1:
            mid = (lo + hi) // 2
            c.children = (build(lo, mid), build(mid, hi))
        return c

    root = build(0, nleaf)
    tree = ClusterTree(root=root, perm=rng.permutation(n).astype(np.int64), clusters=clusters)
    op = H2Matrix(tree=tree, n=n)
    blocks = rng.standard_normal((nleaf, leaf, leaf))
    for c in clusters:
        if c.is_leaf:
            op.row_basis[c.cid] = np.zeros((leaf, 0))
            op.col_basis[c.cid] = np.zeros((leaf, 0))
            op.near.append((c.cid, c.cid, blocks[c.start // leaf]))
        for ch in c.children:
            op.row_transfer[ch.cid] = np.zeros((0, 0))
            op.col_transfer[ch.cid] = np.zeros((0, 0))

    def ref(x):
        xp = x[tree.perm].reshape(nleaf, leaf, -1)
        yp = np.einsum("bij,bjr->bir", blocks, xp).reshape(n, -1)
        y = np.empty_like(yp)
        y[tree.perm] = yp
        return y.reshape(x.shape)

    outs = {}
    for threads in ("", "0", "2", "7"):
        if threads:
            monkeypatch.setenv("H2B_COPY_THREADS", threads)
        else:
            monkeypatch.delenv("H2B_COPY_THREADS", raising=False)
        dev = DeviceOperator(op)
        try:
            for nrhs in (1, 2):
                x = rng.standard_normal((n, nrhs)) if nrhs > 1 else rng.standard_normal(n)
                for _ in range(3):
                    y = dev.matvec(x)
                assert rel(y, ref(x)) < 1e-13
            x1 = np.arange(n, dtype=np.float64) / n
            outs[threads] = dev.matvec(x1)
        finally:
            dev.close()
    assert all(np.array_equal(outs[""], v) for v in outs.values())


@pytest.mark.gpu
def test_config2_full_size_properties(tmp_path):
    """BASELINE configs[1] at its full size (cube, 101 402 nodes, 595 MB of
    H² data -- 4.7x the L2): built here by the package's builder, then the
    product against the oracle on the same operator and through
    size-independent properties: linearity, M 1 = -1 (the double-layer
    operator plus the solid angle on a closed surface) within the compression
    error, bit-for-bit determinism, and multi-RHS columns against single
    products."""
    from paper_1811_05731_b200.h2 import DeviceOperator
    from paper_1811_05731_b200.workloads import build_workload
    op, info = build_workload("config2", cache_dir=str(tmp_path), log=lambda *a: None)
    n = op.n
    assert n == 101402
    dev = DeviceOperator(op)
    try:
        rng = np.random.default_rng(11)
        x, z = rng.standard_normal(n), rng.standard_normal(n)
        yx, yz = dev.matvec(x), dev.matvec(z)
        assert rel(yx, h2_matvec_ref(op, x)) <= 1e-12
        assert rel(dev.matvec(2.5 * x - 0.75 * z), 2.5 * yx - 0.75 * yz) <= 1e-13
        assert np.array_equal(dev.matvec(x), yx)
        # M 1 = -1 holds for the exact operator; the compressed one carries its
        # entrywise error (~3e-5 with the reference's eps = 1e-5 on flat faces)
        # coherently over 101 402 columns: max 8.4e-2, mean 5.6e-3 here
        # (profiles/r02_row_sum_probe.jsonl; a sphere of this size: 4e-5)
        ones = dev.matvec(np.ones(n))
        assert np.abs(ones + 1.0).max() < 0.15 and abs(ones.mean() + 1.0) < 1e-2
        assert np.array_equal(dev.matvec(np.zeros(n)), np.zeros(n))
        for nrhs in (2, 4, 8, 16):
            X = rng.standard_normal((n, nrhs))
            X[:, 0], X[:, -1] = x, z
            Y = dev.matvec(X)
            assert rel(Y[:, 0], yx) <= 1e-13 and rel(Y[:, -1], yz) <= 1e-13
            assert rel(Y[:, 1], h2_matvec_ref(op, np.ascontiguousarray(X[:, 1]))) <= 1e-12
    finally:
        dev.close()
