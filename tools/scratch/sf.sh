#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python tools/sweep.py --config config3 --steps 20 --grid '{"sched_flags": [304611464, 306708616, 310902920, 438829192, 440926344, 445120648, 505938056, 508035208, 512229512], "task_bytes": [262144], "far_task_bytes": [8192]}' --nrhs 1 > gpurun_out/sf_c3.jsonl 2> gpurun_out/sf_c3.err; echo "c3 rc=$?"; cut -c1-190 gpurun_out/sf_c3.jsonl; tail -3 gpurun_out/sf_c3.err | cut -c1-300
