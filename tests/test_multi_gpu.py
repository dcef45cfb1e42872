"""Multi-GPU product: per-rank plans over byte-balanced leaf
ranges, phase 0 (owned x^) -> all-gather of the x^ regions -> phase 1.

* CPU: every rank's plan is executed by the numpy interpreter with an
  emulated all-gather, for 2..8 ranks, golden and adversarial operators;
* CPU, 2 processes over torch.distributed (gloo): the exchange is a real
  collective between processes, as NCCL does it on the GPUs;
* GPU: the ranks run one after another on one device (phase 0 of every
  rank, region copies, phase 1 of every rank) — no kernel ever waits on
  another launch, so this is safe on a single GPU.
"""

import os
import socket
import subprocess
import sys
import textwrap

import numpy as np
import pytest

from conftest import ROOT, load_golden, rel
from oracle.flat_matvec import run_ranks
from oracle.h2_matvec_ref import h2_matvec_ref
from paper_1811_05731_b200.h2 import plan_view
from synth import random_h2


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_rank_plans_reproduce_reference(golden, world):
    name, op, ex = golden
    plans = [plan_view(op, world_size=world, rank=r) for r in range(world)]
    assert sum(p["stats"]["local_bytes"] for p in plans) >= op.storage_bytes() * 0.5
    for i in (0, 4):
        y = run_ranks(plans, ex["X"][:, i])
        assert rel(y, ex["y_full"][:, i]) <= 1e-13, (name, world, i)


@pytest.mark.parametrize("pct", [-1, 1, 25, 100])
def test_rank_plans_near_field_phase_split(golden, pct):
    """Any share of a rank's near field may run in phase 0 (beside the
    upward pass); the finals of phase 1 read those slots."""
    name, op, ex = golden
    for world in (2, 4):
        plans = [plan_view(op, world_size=world, rank=r, near_phase0_pct=pct) for r in range(world)]
        near0 = sum(int((ph["t_kind"] == 3).sum()) for p in plans for ph in p["phases"] if ph["group"] == 0)
        assert (near0 == 0) == (pct == -1) or not op.near
        y = run_ranks(plans, ex["X"][:, 0])
        assert rel(y, ex["y_full"][:, 0]) <= 1e-13, (name, world, pct)


@pytest.mark.parametrize("seed", range(3))
def test_rank_plans_random_structures(seed):
    op = random_h2(seed)
    x = np.random.default_rng(seed).standard_normal(op.n)
    ref = h2_matvec_ref(op, x)
    for world in (2, 5):
        plans = [plan_view(op, world_size=world, rank=r) for r in range(world)]
        assert rel(run_ranks(plans, x), ref) <= 1e-13


def test_partition_is_balanced_and_covers():
    op, _ = load_golden("config1_sphere4")
    world = 4
    plans = [plan_view(op, world_size=world, rank=r) for r in range(world)]
    lohi = plans[0]["rank_lo_hi"]
    assert lohi[0, 0] == 0 and lohi[-1, 1] == op.n
    assert np.all(lohi[1:, 0] == lohi[:-1, 1])
    loads = np.array([p["stats"]["local_bytes"] for p in plans], float)
    assert loads.max() / loads.mean() < 1.25


def test_rank_validation():
    op, _ = load_golden("sphere2_default")
    with pytest.raises(ValueError, match="rank"):
        plan_view(op, world_size=2, rank=2)


_GLOO_WORKER = textwrap.dedent("""
    import os, sys
    import numpy as np
    import torch
    import torch.distributed as dist
    sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
    from conftest import load_golden
    from oracle.flat_matvec import run_group
    from paper_1811_05731_b200.h2 import plan_view
    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:{port}",
                            rank=int(sys.argv[1]), world_size=2)
    r, W = dist.get_rank(), dist.get_world_size()
    op, ex = load_golden("config1_sphere4")
    p = plan_view(op, world_size=W, rank=r)
    x = ex["X"][:, 0]
    coef = np.full((p["coef_len"], 1), np.nan)
    y = np.zeros((op.n, 1))
    run_group(p, 0, x, coef, y)
    off, cnt = p["exchange"]
    parts = [torch.zeros(cnt, dtype=torch.float64) for _ in range(W)]
    dist.all_gather(parts, torch.from_numpy(coef[off + r * cnt: off + (r + 1) * cnt, 0].copy()))
    for q in range(W):
        coef[off + q * cnt: off + (q + 1) * cnt, 0] = parts[q].numpy()
    run_group(p, 1, x, coef, y)
    lo, hi = p["rank_lo_hi"][r]
    mine = np.zeros(op.n)
    mine[p["perm"][lo:hi]] = y[p["perm"][lo:hi], 0]
    t = torch.from_numpy(mine)
    dist.all_reduce(t)
    if r == 0:
        ref = ex["y_full"][:, 0]
        err = np.linalg.norm(t.numpy() - ref) / np.linalg.norm(ref)
        print("REL_ERR", err)
        assert err <= 1e-13
    dist.destroy_process_group()
""")


def test_two_processes_gloo(tmp_path):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    script = tmp_path / "worker.py"
    script.write_text(_GLOO_WORKER.format(root=str(ROOT), tests=str(ROOT / "tests"), port=port))
    env = dict(os.environ, OMP_NUM_THREADS="1")
    procs = [subprocess.Popen([sys.executable, str(script), str(r)], stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT, env=env) for r in range(2)]
    outs = []
    for pr in procs:
        out, _ = pr.communicate(timeout=300)
        outs.append(out.decode())
        assert pr.returncode == 0, out.decode()[-2000:]
    assert "REL_ERR" in outs[0]


# the streaming defaults a large rank operator gets, forced
STREAMING = dict(sched_flags=8 | (8 << 4) | (2 << 18) | (6 << 26) | (4 << 20), far_task_bytes=8192, task_bytes=262144)


@pytest.mark.gpu
@pytest.mark.parametrize("opts", [{}, STREAMING, dict(plan_flags=1 << 8), dict(STREAMING, plan_flags=(1 << 8) | 1)])
@pytest.mark.parametrize("world", [2, 4])
def test_virtual_ranks_on_one_gpu(world, opts):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    from paper_1811_05731_b200.h2 import DeviceOperator
    for name in ("config1_sphere4", "prism_20_40_2_default"):
        op, ex = load_golden(name)
        devs = [DeviceOperator(op, world_size=world, rank=r, **opts) for r in range(world)]
        x = torch.from_numpy(ex["X"][:, 0]).cuda()
        ys = [torch.zeros_like(x) for _ in range(world)]
        s = torch.cuda.current_stream().cuda_stream
        for _ in range(2):  # twice: the per-phase scheduler state must reset
            for r, d in enumerate(devs):
                d.matvec_phase(0, x.data_ptr(), ys[r].data_ptr(), 1, s)
            for r, d in enumerate(devs):
                for q, o in enumerate(devs):
                    if q != r:
                        d.exchange_copy_from(o, 1, s)
            for r, d in enumerate(devs):
                d.matvec_phase(1, x.data_ptr(), ys[r].data_ptr(), 1, s)
            torch.cuda.synchronize()
            plans = [plan_view(op, world_size=world, rank=r, **opts) for r in range(world)]
            y = np.zeros(op.n)
            for r in range(world):
                lo, hi = plans[r]["rank_lo_hi"][r]
                rows = plans[r]["perm"][lo:hi]
                y[rows] = ys[r].cpu().numpy()[rows]
            assert rel(y, ex["y_full"][:, 0]) <= 1e-12, (name, world)
        for d in devs:
            d.close()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_rank_pool_holds_only_selected_items(golden, world):
    """Per-rank storage (VERDICT r1 task 5): a rank's matrix pool is exactly
    the bytes of the items it runs (its rows plus the replicated upper
    clusters), so per-rank host and device memory scale as 1/world."""
    name, op, ex = golden
    full = plan_view(op)["stats"]["pool_bytes"]
    pools = []
    for r in range(world):
        st = plan_view(op, world_size=world, rank=r)["stats"]
        assert st["pool_bytes"] == st["local_bytes"], (name, world, r)
        pools.append(st["pool_bytes"])
    assert sum(pools) >= full                      # every matrix is somewhere
    assert max(pools) < full or world > len(op.tree.clusters) // 2
    # replication (upper clusters spanning ranks) stays a small part
    assert sum(pools) <= 1.25 * full + 8 * 4096 * world, (name, world, sum(pools) / full)
