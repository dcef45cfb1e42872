"""H2MS operator files: the native reader/writer against
files written by the reference's own save_h2 (tests/golden/make_h2ms.py),
and the reference's persistence tests restated (test_hmatrix.py:345-394)."""

import os
import struct

import numpy as np
import pytest

from conftest import GOLDEN, load_golden, rel
from oracle.h2_matvec_ref import h2_matvec_ref
from paper_1811_05731_b200.persist import (H2MSFile, OperatorIOError, crc64, load_device_operator, load_h2,
                                           save_h2)

REF_FILE = GOLDEN / "sphere2_default.h2ms"


def _same_operator(a, b):
    assert a.n == b.n
    assert np.array_equal(a.tree.perm, b.tree.perm)
    assert len(a.tree.clusters) == len(b.tree.clusters)
    for ca, cb in zip(a.tree.clusters, b.tree.clusters):
        assert (ca.start, ca.end, ca.cid, ca.is_leaf) == (cb.start, cb.end, cb.cid, cb.is_leaf)
        assert np.array_equal(ca.bbox_min, cb.bbox_min) and np.array_equal(ca.bbox_max, cb.bbox_max)
    for d in ("row_basis", "col_basis", "row_transfer", "col_transfer"):
        da, db = getattr(a, d), getattr(b, d)
        assert sorted(da) == sorted(db), d
        for k in da:
            assert np.array_equal(da[k], db[k]), (d, k)
    for la, lb in ((a.coupling, b.coupling), (a.near, b.near)):
        assert len(la) == len(lb)
        for (r1, c1, m1), (r2, c2, m2) in zip(la, lb):
            assert (r1, c1) == (r2, c2) and np.array_equal(m1, m2)


def test_crc64_reference_vector():
    # CRC-64/XZ check value for the ASCII digits "123456789" (test_hmatrix.py:392-394)
    assert crc64(b"123456789") == 0x995DC9BBDF1939FA
    assert crc64(b"") == 0


def _crc_py(data: bytes) -> int:
    """Bytewise table CRC-64/XZ, as persist.py:24-38 states it."""
    poly, tab = 0xC96C5795D7870F42, []
    for b in range(256):
        c = b
        for _ in range(8):
            c = (c >> 1) ^ poly if c & 1 else c >> 1
        tab.append(c)
    crc = 0xFFFFFFFFFFFFFFFF
    for x in data:
        crc = tab[(crc ^ x) & 0xFF] ^ (crc >> 8)
    return crc ^ 0xFFFFFFFFFFFFFFFF


def test_crc64_matches_bytewise_and_threads_combine(monkeypatch):
    rng = np.random.default_rng(7)
    for n in (1, 7, 8, 9, 1000, 65537):
        b = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        assert crc64(b) == _crc_py(b)
    big = rng.integers(0, 256, 40 * 2**20 + 13, dtype=np.uint8).tobytes()
    multi = crc64(big)                       # split over host threads, joined by CRC combination
    monkeypatch.setenv("H2B_CRC_THREADS", "1")
    assert crc64(big) == multi


def test_reference_file_loads_to_the_same_operator():
    op_ref, ex = load_golden("sphere2_default")
    loaded = load_h2(REF_FILE, expected_n=op_ref.n)
    _same_operator(loaded, op_ref)
    assert loaded.storage_bytes() == int(ex["storage_bytes"])
    for i in range(3):
        assert np.array_equal(h2_matvec_ref(loaded, ex["X"][:, i]), ex["y_full"][:, i])


def test_writer_is_byte_identical_to_the_reference(tmp_path):
    op = load_h2(REF_FILE)
    out = tmp_path / "op.h2m"
    save_h2(op, out)
    assert out.read_bytes() == REF_FILE.read_bytes()


@pytest.mark.parametrize("name", ["sphere3_l32_eta2_o4", "torus_32_16_4_default"])
def test_roundtrip(name, tmp_path):
    op, ex = load_golden(name)
    path = tmp_path / "op.h2m"
    save_h2(op, path)
    back = load_h2(path, expected_n=op.n)
    _same_operator(back, op)
    assert np.array_equal(h2_matvec_ref(back, ex["X"][:, 0]), h2_matvec_ref(op, ex["X"][:, 0]))


def test_checksum_mismatch(tmp_path):
    data = bytearray(REF_FILE.read_bytes())
    data[len(data) // 2] ^= 0x01
    p = tmp_path / "op.h2m"
    p.write_bytes(bytes(data))
    with pytest.raises(OperatorIOError, match="checksum"):
        load_h2(p)


def test_truncated_file(tmp_path):
    p = tmp_path / "op.h2m"
    p.write_bytes(REF_FILE.read_bytes()[:50])
    with pytest.raises(OperatorIOError):
        load_h2(p)
    p.write_bytes(REF_FILE.read_bytes()[:10])
    with pytest.raises(OperatorIOError, match="truncated"):
        load_h2(p)


def _with_crc(body: bytes) -> bytes:
    return body + struct.pack("<Q", crc64(body))


def test_bad_magic(tmp_path):
    p = tmp_path / "op.h2m"
    p.write_bytes(_with_crc(b"XXXX" + REF_FILE.read_bytes()[4:-8]))
    with pytest.raises(OperatorIOError, match="magic"):
        load_h2(p)


def test_unsupported_version(tmp_path):
    body = REF_FILE.read_bytes()[:-8]
    p = tmp_path / "op.h2m"
    p.write_bytes(_with_crc(body[:4] + struct.pack("<I", 2) + body[8:]))
    with pytest.raises(OperatorIOError, match="version 2"):
        load_h2(p)


def test_trailing_garbage(tmp_path):
    p = tmp_path / "op.h2m"
    p.write_bytes(_with_crc(REF_FILE.read_bytes()[:-8] + b"\0"))
    with pytest.raises(OperatorIOError, match="trailing garbage"):
        load_h2(p)


def test_node_count_mismatch():
    with pytest.raises(OperatorIOError, match="boundary nodes"):
        load_h2(REF_FILE, expected_n=163)


def test_missing_file(tmp_path):
    with pytest.raises(OperatorIOError):
        load_h2(tmp_path / "nope.h2m")


def test_file_descriptor_plans_like_the_operator():
    """The descriptor view of an opened file is what h2b_create consumes: its
    plan must equal the plan of the in-memory operator."""
    from paper_1811_05731_b200 import _native as nat
    from paper_1811_05731_b200.h2 import plan_view
    import ctypes as C
    op, _ = load_golden("sphere2_default")
    ref = plan_view(op)
    with H2MSFile(REF_FILE) as f:
        lib = nat.lib()
        h = C.c_void_p()
        from paper_1811_05731_b200.h2 import _options
        nat.check(lib.h2b_plan_create(C.byref(f.desc), C.byref(_options()), C.byref(h)))
        try:
            v = nat.PlanView()
            nat.check(lib.h2b_plan_view_get(h, C.byref(v)))
            mat = np.ctypeslib.as_array(v.mat, shape=(v.mat_len,)).copy()
        finally:
            lib.h2b_plan_destroy(h)
    assert np.array_equal(mat, ref["mat"])


@pytest.mark.gpu
def test_file_straight_to_device():
    op, ex = load_golden("sphere2_default")
    dev = load_device_operator(REF_FILE, expected_n=op.n)
    try:
        for i in range(3):
            assert rel(dev.matvec(ex["X"][:, i]), ex["y_full"][:, i]) <= 1e-12
        assert dev.stream_bytes() == int(ex["storage_bytes"])
    finally:
        dev.close()


def test_workload_cache_roundtrip_memory_mapped(tmp_path):
    """bench.py's operator cache (one .npy per array, memory-mapped on load)
    returns the same operator and the same product."""
    from oracle.h2_matvec_ref import h2_matvec_ref
    from paper_1811_05731_b200.workloads import load_cached, save_cached
    op, ex = load_golden("torus_32_16_4_default")
    save_cached(op, tmp_path / "op")
    op2 = load_cached(tmp_path / "op")
    assert op2.n == op.n and op2.storage_bytes() == op.storage_bytes()
    assert isinstance(op2.near[0][2].base, np.memmap) or isinstance(op2.near[0][2], np.memmap) \
        or op2.near[0][2].flags["OWNDATA"] is False
    x = ex["X"][:, 0]
    assert np.array_equal(h2_matvec_ref(op2, x), h2_matvec_ref(op, x))
