#!/bin/bash
mkdir -p gpurun_out
ls /tmp/h2b_cache 2>/dev/null; df -h /tmp | tail -1
# unit sizes of the sweeps: default (16384 nodes, 256 units), 8192, 4096
timeout 2400 python tools/sweep.py --config config5 --steps 10 --grid '{"plan_flags":[0,29696,25600]}' > gpurun_out/c5_units.jsonl 2> gpurun_out/c5_units.err; echo "sweep rc=$?"; cut -c1-150 gpurun_out/c5_units.jsonl; tail -2 gpurun_out/c5_units.err | cut -c1-300
timeout 1500 python tools/rank_sim.py --config config5 --worlds 2,4,8 --steps 10 --modes "" --defaults > gpurun_out/c5_ranksim2.jsonl 2> gpurun_out/c5_ranksim2.err; echo "ranksim rc=$?"; cut -c1-330 gpurun_out/c5_ranksim2.jsonl
