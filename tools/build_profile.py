"""Time the operator build of a surface with a given backend (no cache).

    python tools/build_profile.py --config config2 --backend gpu"""

import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="config2")
    ap.add_argument("--backend", default="gpu")
    a = ap.parse_args()
    import __graft_entry__
    __graft_entry__.build()
    from paper_1811_05731_b200.assembly.hbuild import assemble_h2
    from paper_1811_05731_b200.workloads import WORKLOADS
    w = WORKLOADS[a.config]
    t = time.perf_counter()
    surf = w["surface"]()
    print(f"surface {surf.n} ({time.perf_counter() - t:.1f}s)", flush=True)
    op, rep = assemble_h2(surf, w["cfg"], backend=a.backend, log=lambda m: print(m, flush=True))
    print({k: round(v, 2) for k, v in rep.seconds.items()}, op.storage_bytes())


if __name__ == "__main__":
    main()
