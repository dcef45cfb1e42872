#!/bin/bash
# config 3 built with the GPU recompression: build log, bench with operator check; then the host-recompressed one for comparison
mkdir -p gpurun_out
H2B_RECOMPRESS=gpu timeout 1500 python bench.py --config config3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/rc3_bench_gpu.json 2> gpurun_out/rc3_bench_gpu.err; echo "gpu-rec bench rc=$?"
grep -i "recompress\|operator check\|parity\|HCA (gpu)" gpurun_out/rc3_bench_gpu.err | cut -c1-400
cut -c1-200 gpurun_out/rc3_bench_gpu.json
timeout 1500 python bench.py --config config3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/rc3_bench_host.json 2> gpurun_out/rc3_bench_host.err; echo "host-rec bench rc=$?"
grep -i "recompress\|operator check\|parity" gpurun_out/rc3_bench_host.err | cut -c1-400
cut -c1-200 gpurun_out/rc3_bench_host.json
