#!/bin/bash
mkdir -p gpurun_out
MEMGUARD_MIN_KB=12000000 tools/memguard.sh gpurun_out/c5_guard.log python bench.py --config config5 --steps 10 --warmup 3 > gpurun_out/c5_bench.json 2> gpurun_out/c5_bench.err; echo "bench rc=$?"
tail -2 gpurun_out/c5_guard.log
cut -c1-300 gpurun_out/c5_bench.json
timeout 900 python tools/sweep.py --config config5 --steps 10 --grid '{"plan_flags":[2048,0]}' > gpurun_out/c5_sweep.jsonl 2> gpurun_out/c5_sweep.err; echo "sweep rc=$?"; cut -c1-150 gpurun_out/c5_sweep.jsonl
timeout 1200 python tools/rank_sim.py --config config5 --worlds 8 --steps 10 --modes "" --defaults --plan-flags 0,2048 > gpurun_out/c5_ranksim.jsonl 2> gpurun_out/c5_ranksim.err; echo "ranksim rc=$?"; cut -c1-300 gpurun_out/c5_ranksim.jsonl
for ph in 0 1 2; do timeout 600 python tools/trace.py --config config5 --phase $ph > gpurun_out/c5_trace_$ph.txt 2>&1; done
grep -v workload gpurun_out/c5_trace_1.txt | cut -c1-200 | head -20
