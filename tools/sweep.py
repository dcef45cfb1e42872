"""Time the H² product of a workload under several plan/launch options.

    python tools/sweep.py --config config2 [--steps 100]

Prints one line per option set: ms per product, GB/s of algorithmic bytes.
Used to choose defaults; bench.py reports the chosen configuration."""

import argparse
import itertools
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="config2")
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--cache-dir", default="/tmp/h2b_cache")
    ap.add_argument("--grid", default='{"task_bytes":[16384,32768,65536],"interleave":[0,-1]}')
    ap.add_argument("--flush", action="store_true", help="flush L2 before each timed step")
    ap.add_argument("--nrhs", default="1", help="comma list of right-hand-side counts")
    ap.add_argument("--ablate", default="", help="comma list of: far (near=[]), near (coupling=[])")
    ap.add_argument("--env", default="[{}]", help='JSON list of environment settings read at create, '
                                                  'e.g. [{"H2B_NEAR_SPLIT":"0"},{}]')
    a = ap.parse_args()
    import torch
    import __graft_entry__
    __graft_entry__.build()
    from paper_1811_05731_b200.h2 import DeviceOperator
    from paper_1811_05731_b200.workloads import build_workload, vector_for
    op, _ = build_workload(a.config, cache_dir=a.cache_dir, log=lambda m: print(m, file=sys.stderr))
    import dataclasses
    ops = {"full": op}
    for ab in filter(None, a.ablate.split(",")):
        ops[ab] = dataclasses.replace(op, near=[]) if ab == "far" else dataclasses.replace(op, coupling=[])
    grid = json.loads(a.grid)
    keys = list(grid)
    s = torch.cuda.current_stream()
    nrhs_list = [int(v) for v in a.nrhs.split(",")]
    from bench import DeviceTimer
    timer = DeviceTimer(s, flush=a.flush)
    refs = {}
    import os
    envs = json.loads(a.env)
    for (name, opx), nrhs, vals, env in itertools.product(ops.items(), nrhs_list,
                                                          itertools.product(*[grid[k] for k in keys]), envs):
        opts = dict(zip(keys, vals))
        old_env = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        dev = DeviceOperator(opx, **opts)
        for k, v in old_env.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
        st = dev.stats()
        x = torch.from_numpy(np.ascontiguousarray(vector_for(a.config, op.n, nrhs))).cuda()
        y = torch.empty_like(x)
        for _ in range(5):
            dev.matvec_dev(x.data_ptr(), y.data_ptr(), nrhs, s.cuda_stream)
        ms = timer.run(lambda: dev.matvec_dev(x.data_ptr(), y.data_ptr(), nrhs, s.cuda_stream), a.steps)
        yy = y.cpu().numpy()
        ref = refs.setdefault((name, nrhs), yy)
        err = float(np.linalg.norm(yy - ref) / np.linalg.norm(ref))
        gbs = (st["stream_bytes"] + 16 * op.n * nrhs) / (ms * 1e-3) / 1e9
        print(json.dumps({"op": name, "nrhs": nrhs, "opts": opts, "env": env, "ms": round(ms, 4), "GB/s": round(gbs, 1),
                          "ms_per_vector": round(ms / nrhs, 4), "items": st["ntasks"],
                          "grid": st["grid"], "rel_vs_first": err}), flush=True)
        dev.close()


if __name__ == "__main__":
    main()
