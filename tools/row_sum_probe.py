"""How far M 1 is from -1 for H² operators of growing size (diagnostics).

The exact operator satisfies M 1 = -1 on a closed surface (test_bem.py:96-102).
The compressed one does so up to its compression error, which for the
constant vector adds up coherently over the admissible blocks.  Cubes of
q x q quads per face, config 2's parameters (leaf 64, eta 2, order 5), the
reference's thresholds eps = 1e-5 / eps_rec = 2e-4 and tighter ones.

    python tools/row_sum_probe.py 16 32 64 130
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import __graft_entry__
    __graft_entry__.build()
    from paper_1811_05731_b200.assembly import geometry as G
    from paper_1811_05731_b200.assembly.hbuild import CompressionConfig, assemble_h2
    from paper_1811_05731_b200.h2 import DeviceOperator
    for q in [int(a) for a in sys.argv[1:]]:
        s = G.cube_surface(q)
        for eps, eps_rec in ((1e-5, 2e-4), (1e-5, 1e-6), (1e-7, 1e-6)):
            cfg = CompressionConfig(leaf_size=64, eta=2.0, cheb_order=5, eps=eps, eps_rec=eps_rec)
            t = time.time()
            op, rep = assemble_h2(s, cfg, backend="numpy")
            dev = DeviceOperator(op)
            v = dev.matvec(np.ones(op.n))
            x = np.random.default_rng(0).standard_normal(op.n)
            y = dev.matvec(x)
            dev.close()
            print(json.dumps({"q": q, "n": op.n, "eps": eps, "eps_rec": eps_rec,
                              "max_abs_M1_plus_1": float(np.abs(v + 1).max()), "mean_M1_plus_1": float(v.mean() + 1),
                              "rms_y_randn": float(np.sqrt(np.mean(y ** 2))), "h2_mb": op.storage_bytes() / 1e6,
                              "admissible": rep.n_admissible, "seconds": round(time.time() - t, 1)}), flush=True)


if __name__ == "__main__":
    main()
