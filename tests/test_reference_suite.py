"""The reference's own tests, run against the GPU product (SURVEY §4 "How
the new repo should test", VERDICT r1 task 3).

The unmodified reference is imported from ``baseline/_ref`` (installed by
tools/vendor_reference.sh); its tests run in a child pytest with
tests/refsuite/gpu_patch_plugin.py, which installs the GPU ``h2_matvec`` into
the reference module exactly as INTEGRATION.md §1 tells maintainers to, and
counts the products that went through it.  Reference test files:
tests/test_hmatrix.py:254-331 (TestH2), :348-394 (TestPersistence),
tests/test_acceptance.py:80-100 (backend equivalence), :166-188
(persistence round trip and cached rerun).
"""

import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"

SELECTION = [
    "test_hmatrix.py::TestH2",
    "test_hmatrix.py::TestPersistence",
    "test_acceptance.py::test_backend_equivalence",
    "test_acceptance.py::test_persistence_round_trip_and_cached_rerun",
]


def _run(selection, tmp_path, timeout=1500):
    count = tmp_path / "count.txt"
    env = dict(os.environ, H2B_REFSUITE_COUNT=str(count),
               PYTHONPATH=os.pathsep.join([str(ROOT / "tests" / "refsuite"), str(REF), str(ROOT)]))
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-p", "gpu_patch_plugin",
           "-c", str(ROOT / "tests" / "refsuite" / "pytest.ini"), "--rootdir", str(REF / "tests"),
           *[str(REF / "tests" / s) for s in selection]]
    r = subprocess.run(cmd, cwd=str(REF / "tests"), env=env, capture_output=True, text=True, timeout=timeout)
    calls = int(count.read_text()) if count.exists() else -1
    return r, calls


@pytest.mark.skipif(not (REF / "tests" / "test_hmatrix.py").exists(),
                    reason="baseline/_ref not vendored (tools/vendor_reference.sh)")
@pytest.mark.gpu
def test_reference_suite_on_gpu_path(tmp_path):
    r, calls = _run(SELECTION, tmp_path)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, tail
    assert "passed" in r.stdout and "failed" not in r.stdout, tail
    # every H2Matrix.matvec of those tests went through the GPU path
    assert calls >= 100, f"only {calls} products reached the patched h2_matvec\n{tail}"
