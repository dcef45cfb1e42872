import json, sys, time
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
def main():
    import __graft_entry__
    __graft_entry__.build()
    from paper_1811_05731_b200.assembly import geometry as G
    from paper_1811_05731_b200.assembly.hbuild import CompressionConfig, assemble_h2
    from paper_1811_05731_b200.h2 import DeviceOperator
    from paper_1811_05731_b200.workloads import exact_rows
    surfs = {"cube16": G.cube_surface(16), "cube32": G.cube_surface(32), "ico4": G.icosphere_surface(4), "ico5": G.icosphere_surface(5)}
    for name, s in surfs.items():
        ex = exact_rows(s, np.arange(0, s.n, max(1, s.n // 64)))
        rows = np.arange(0, s.n, max(1, s.n // 64))
        for leaf, eta, order in ((32, 3.0, 5), (64, 3.0, 5), (32, 2.0, 5), (64, 2.0, 5), (64, 2.0, 7), (64, 1.0, 5)):
            cfg = CompressionConfig(leaf_size=leaf, eta=eta, cheb_order=order)
            op, rep = assemble_h2(s, cfg, backend="numpy")
            dev = DeviceOperator(op)
            v = dev.matvec(np.ones(op.n))
            # entrywise error of sampled rows: M_h2^T e_i is not available; use unit-vector products for a few columns instead
            cols = rows[:8]
            E = np.stack([dev.matvec(np.eye(1, op.n, int(c))[0]) for c in cols], axis=1)   # columns of M_h2
            exact_cols = exact_rows(s, np.arange(s.n))[:, cols] if s.n <= 3000 else None
            dev.close()
            out = {"surface": name, "n": op.n, "leaf": leaf, "eta": eta, "order": order,
                   "max_abs_M1_plus_1": float(np.abs(v + 1).max()), "admissible": rep.n_admissible, "fallback": rep.n_fallback}
            if exact_cols is not None:
                out["max_entry_err"] = float(np.abs(E - exact_cols).max())
                out["max_entry"] = float(np.abs(exact_cols).max())
            print(json.dumps(out), flush=True)


if __name__ == '__main__':
    main()
