#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "staged_copies" 2>&1 | tail -3
for V in "0 256" "4 256" "8 256" "8 128" "8 512" "12 256"; do set -- $V
H2B_COPY_THREADS=$1 H2B_COPY_CHUNK_KB=$2 timeout 600 python tools/e2e_probe.py --config config3 > gpurun_out/e2e_$1_$2.json 2> gpurun_out/e2e_$1_$2.err; echo "threads $1 chunk $2 KB rc=$?"; cut -c60-400 gpurun_out/e2e_$1_$2.json
done
