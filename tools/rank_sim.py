"""Per-rank time of the sharded product, one rank at a time on one GPU.

    python tools/rank_sim.py --config config3 --worlds 2,4,8 [--steps 30]

For each world size and rank, the rank operator runs its two
phases back to back on the local GPU; the all-gather between them is left
out (its ~N_coef·8 bytes per rank move over NVLink in microseconds), so the
coefficients phase 1 reads are stale -- the work and the bytes are the
same, the values are not checked.  The max over ranks models the step time
of an N-GPU run; ranks never wait on each other here.  Both scheduling
modes are timed (plain, and the streaming defaults forced) to place the
H2B_STREAM_DEFAULT_BYTES threshold.

The all-gather is added back as a modeled term: every rank's exchange
region (x^ of the clusters it owns; h2b_exchange_region) is all-gathered,
W * region * 8 bytes in total, costed at a fixed latency plus that volume
over NVLink 5 (--ag-latency-us, --ag-gbs: NCCL all-gather of small messages
on 8 GPUs behind NVSwitch; not measured here, only one GPU is available).
``modeled_ms = max over ranks (phase 0 + phase 1) + all-gather``."""

import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

STREAMING = dict(sched_flags=8 | (8 << 4) | (2 << 18) | (6 << 26) | (4 << 20) | (1 << 25), far_task_bytes=8192, task_bytes=131072)
PLAIN = dict(sched_flags=8)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="config3")
    ap.add_argument("--worlds", default="2,4,8")
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--cache-dir", default="/tmp/h2b_cache")
    ap.add_argument("--pct", default="0", help="comma list of near_phase0_pct values (0: default)")
    ap.add_argument("--modes", default="plain,streaming")
    ap.add_argument("--defaults", action="store_true", help="also time the library defaults (no forced mode)")
    ap.add_argument("--ag-latency-us", type=float, default=15.0)
    ap.add_argument("--ag-gbs", type=float, default=300.0)
    ap.add_argument("--plan-flags", default="0", help="comma list of h2b_options.plan_flags values")
    a = ap.parse_args()
    import torch
    import __graft_entry__
    __graft_entry__.build()
    from paper_1811_05731_b200.h2 import DeviceOperator
    from paper_1811_05731_b200.workloads import build_workload, vector_for
    op, _ = build_workload(a.config, cache_dir=a.cache_dir, log=lambda m: print(m, file=sys.stderr))
    x = torch.from_numpy(vector_for(a.config, op.n)).cuda()
    y = torch.zeros_like(x)
    s = torch.cuda.current_stream()
    for world in [int(w) for w in a.worlds.split(",")]:
        modes = [(m, dict(PLAIN if m == "plain" else STREAMING, near_phase0_pct=int(pc), plan_flags=int(pf)))
                 for m in filter(None, a.modes.split(",")) for pc in a.pct.split(",")
                 for pf in a.plan_flags.split(",")]
        if a.defaults:
            modes += [("defaults", dict(near_phase0_pct=0, plan_flags=int(pf))) for pf in a.plan_flags.split(",")]
        for mode, opts in modes:
            per_rank = []
            exch = 0
            for r in range(world):
                dev = DeviceOperator(op, world_size=world, rank=r, **opts)
                st = dev.stats()
                exch = dev.exchange_region(1)[1] if world > 1 else 0
                phases = 1 if world == 1 else 2
                run = lambda: [dev.matvec_phase(k, x.data_ptr(), y.data_ptr(), 1, s.cuda_stream)
                               for k in range(phases)]
                for _ in range(3):
                    run()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                for _ in range(a.steps):
                    run()
                e1.record(s)
                torch.cuda.synchronize()
                per_rank.append((e0.elapsed_time(e1) / a.steps, int(st["local_bytes"])))
                dev.close()
            t = max(p[0] for p in per_rank)
            ag_bytes = 8 * exch * world
            ag_ms = 0.0 if world == 1 else (a.ag_latency_us + ag_bytes / (a.ag_gbs * 1e3)) / 1e3
            print(json.dumps({"config": a.config, "world": world, "mode": mode,
                              "near_phase0_pct": opts["near_phase0_pct"], "plan_flags": opts.get("plan_flags", 0),
                              "max_rank_ms": round(t, 4),
                              "allgather_bytes": ag_bytes, "allgather_ms_modeled": round(ag_ms, 4),
                              "modeled_ms": round(t + ag_ms, 4),
                              "modeled_DOF_per_s_with_allgather": op.n / ((t + ag_ms) * 1e-3),
                              "rank_ms": [round(p[0], 4) for p in per_rank],
                              "rank_bytes": [p[1] for p in per_rank],
                              "modeled_DOF_per_s": op.n / (t * 1e-3)}), flush=True)


if __name__ == "__main__":
    main()
