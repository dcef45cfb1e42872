#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/sweep.py --config config3 --steps 30 --grid '{}' --env '[{"H2B_SWEEP_PREFETCH":"0"},{"H2B_SWEEP_PREFETCH":"1"},{"H2B_SWEEP_PREFETCH":"2"},{"H2B_SWEEP_PREFETCH":"4"},{"H2B_SWEEP_PREFETCH":"3"},{"H2B_SWEEP_PREFETCH":"0"},{"H2B_SWEEP_PREFETCH":"1"}]' > gpurun_out/pf_c3.jsonl 2> gpurun_out/pf_c3.err; echo "c3 rc=$?"; cut -c1-160 gpurun_out/pf_c3.jsonl
