#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python tools/sweep.py --config config3 --steps 20 --grid '{"task_bytes":[131072,196608,262144,393216]}' --nrhs 1,8,16 > gpurun_out/tb_c3.jsonl 2> gpurun_out/tb_c3.err; echo "c3 rc=$?"; cut -c1-150 gpurun_out/tb_c3.jsonl; tail -3 gpurun_out/tb_c3.err | cut -c1-300
