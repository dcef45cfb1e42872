for v in 4 5; do H2B_CG_VARIANT=$v timeout 600 python -m pytest tests/test_fem_gpu.py -m gpu -x -q 2>&1 | tail -1 | sed "s/^/v$v /" >> gpurun_out/cg_tests4.log; done
for v in 0 4 5 0 4 5; do
  H2B_CG_VARIANT=$v timeout 300 python tools/cg_bench.py --n 96 --reps 9 | sed "s/^/v$v /" >> gpurun_out/cg_sweep4.log 2>&1
done
for v in 0 4 5; do H2B_CG_VARIANT=$v timeout 300 python tools/cg_bench.py --n 48 --reps 9 | sed "s/^/v$v /" >> gpurun_out/cg_sweep4.log 2>&1; done
for v in 0 4 5; do H2B_CG_VARIANT=$v timeout 300 python tools/cg_bench.py --n 160 --reps 3 | sed "s/^/v$v /" >> gpurun_out/cg_sweep4.log 2>&1; done
