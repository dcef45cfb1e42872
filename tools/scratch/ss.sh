#!/bin/bash
mkdir -p gpurun_out
H2B_SPLIT_SWEEPS=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_staged.py -m gpu -x -q -k "rhs or multi" 2>&1 | tail -4
timeout 1200 python tools/sweep.py --config config3 --steps 20 --grid '{}' --nrhs 8,16 --env '[{"H2B_SPLIT_SWEEPS":"0"},{"H2B_SPLIT_SWEEPS":"1"},{"H2B_SPLIT_SWEEPS":"0"},{"H2B_SPLIT_SWEEPS":"1"}]' > gpurun_out/ss_c3.jsonl 2> gpurun_out/ss_c3.err; echo "c3 rc=$?"; cut -c1-200 gpurun_out/ss_c3.jsonl; tail -3 gpurun_out/ss_c3.err | cut -c1-300
