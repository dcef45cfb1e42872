#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "rhs or multi" > gpurun_out/mrhs_test.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/mrhs_test.log
timeout 1200 python tools/sweep.py --config config3 --steps 20 --grid '{}' --nrhs 8,16 --env '[{"H2B_MRHS_SRC_IN_STAGE":"0"},{"H2B_MRHS_SRC_IN_STAGE":"1"},{"H2B_MRHS_SRC_IN_STAGE":"0"},{"H2B_MRHS_SRC_IN_STAGE":"1"}]' > gpurun_out/mrhs_c3.jsonl 2> gpurun_out/mrhs_c3.err; echo "c3 rc=$?"; cut -c1-200 gpurun_out/mrhs_c3.jsonl
