"""Operator files written by the REFERENCE's own ``save_h2``
(hmatrix/persist.py:117-135), for the H2MS reader/writer parity tests.

Run in the build container only (imports /root/reference/pkg/src):

    python tests/golden/make_h2ms.py

Writes ``sphere2_default.h2ms``: the sphere-level-2 operator with the
code-default CompressionConfig (the fixture of the reference's persistence
tests, test_hmatrix.py:345-394), the same operator as sphere2_default.npz.
"""

from __future__ import annotations

import sys
from pathlib import Path

REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

from strayfield import hmatrix as hm  # noqa: E402
from strayfield import mesh as meshmod  # noqa: E402


def main() -> None:
    mesh = meshmod.generate_sphere_mesh(1.0, 2)
    op = hm.assemble_operator(mesh, "h2", hm.CompressionConfig()).payload
    path = HERE / "sphere2_default.h2ms"
    hm.save_h2(op, path)
    print(f"{path.name}: n={op.n} bytes={path.stat().st_size}")


if __name__ == "__main__":
    main()
