"""Write tests/golden/<config>_structure.npz: the per-cluster ranks and
storage_bytes of a workload's operator, from which oracle/reference.py
``structure_twin`` rebuilds an operator of identical structure on the host
(the reference arm of bench.py).  Run where the operator is built (the GPU
box for configs 2-5), e.g.

    python tools/structure_fixture.py --config config3 --out gpurun_out/
    python tools/structure_fixture.py --config config1 --from-npz tests/golden/config1_sphere4.npz
"""

import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", required=True)
    ap.add_argument("--from-npz", default=None)
    ap.add_argument("--cache-dir", default="/tmp/h2b_cache")
    ap.add_argument("--out", default=str(ROOT / "tests" / "golden"))
    a = ap.parse_args()
    from paper_1811_05731_b200.h2 import rank_arrays
    if a.from_npz:
        from paper_1811_05731_b200.io import load_npz
        op, _ = load_npz(a.from_npz)
    else:
        import __graft_entry__
        __graft_entry__.build()
        from paper_1811_05731_b200.workloads import build_workload
        op, _ = build_workload(a.config, cache_dir=a.cache_dir, log=lambda m: print(m, flush=True))
    k_row, k_col = rank_arrays(op)
    out = Path(a.out) / f"{a.config}_structure.npz"
    np.savez_compressed(out, k_row=k_row.astype(np.int32), k_col=k_col.astype(np.int32), n=np.int64(op.n),
                        n_admissible=np.int64(len(op.coupling)), n_near=np.int64(len(op.near)),
                        storage_bytes=np.int64(op.storage_bytes()))
    print(f"wrote {out}: n={op.n} storage_bytes={op.storage_bytes()}")


if __name__ == "__main__":
    main()
