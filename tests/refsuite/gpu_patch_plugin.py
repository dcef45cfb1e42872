"""pytest plugin: run the REFERENCE's own test suite with its H² matvec
routed to the GPU path (test infrastructure).

Loaded with ``-p gpu_patch_plugin`` by tests/test_reference_suite.py in a
child pytest whose rootdir is ``baseline/_ref/tests``.  At configure time it
imports the unmodified reference from ``baseline/_ref`` and calls
``paper_1811_05731_b200.h2.install_into_reference`` on
``strayfield.hmatrix.h2`` and ``strayfield.hmatrix`` (the switch
INTEGRATION.md §1 gives maintainers: ``H2Matrix.matvec`` looks the
module-global up at call time, h2.py:74-75).  A counting wrapper records
how many products went through the GPU path; the count is written to
$H2B_REFSUITE_COUNT at session end.
"""

import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
_count = {"calls": 0}


def pytest_configure(config):
    sys.path.insert(0, str(ROOT))
    from oracle.reference import strayfield
    strayfield()
    import strayfield.hmatrix as hm
    import strayfield.hmatrix.h2 as h2m
    from paper_1811_05731_b200 import h2 as gpu
    gpu.install_into_reference(h2m, hm)
    assert h2m.h2_matvec is gpu.h2_matvec and hm.h2_matvec is gpu.h2_matvec

    def counted(op, x):
        _count["calls"] += 1
        return gpu.h2_matvec(op, x)

    h2m.h2_matvec = counted
    hm.h2_matvec = counted


def pytest_unconfigure(config):
    out = os.environ.get("H2B_REFSUITE_COUNT")
    if out:
        Path(out).write_text(str(_count["calls"]))
