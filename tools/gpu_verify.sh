#!/bin/bash
# Round-end style verification on one B200: GPU tests, smoke, default bench,
# ncu launch list and full captures of the dataflow and sweep kernels.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "gputest rc=$?"; tail -3 gpurun_out/gputest.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --profile > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:h2b_dataflow_kernel -s 3 -c 1 -o gpurun_out/dataflow_full python bench.py --steps 2 --warmup 3 --profile > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:h2b_sweep -s 6 -c 2 -o gpurun_out/sweep_full python bench.py --steps 2 --warmup 3 --profile > gpurun_out/ncu_sweep.log 2>&1; echo "ncu sweep rc=$?"
# the other BASELINE configurations (short runs): config 4 = config 3 with 16 right-hand sides, config 2, config 1
timeout 900 python bench.py --config config3 --nrhs 16 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_config4.json 2> gpurun_out/bench_config4.err; echo "config4 rc=$?"; cut -c1-300 gpurun_out/bench_config4.json
timeout 900 python bench.py --config config2 --steps 50 --warmup 5 > gpurun_out/bench_config2.json 2> gpurun_out/bench_config2.err; echo "config2 rc=$?"; cut -c1-300 gpurun_out/bench_config2.json
timeout 900 python bench.py --config config1 --steps 100 --warmup 5 > gpurun_out/bench_config1.json 2> gpurun_out/bench_config1.err; echo "config1 rc=$?"; cut -c1-300 gpurun_out/bench_config1.json
timeout 900 python bench.py --impl reference --steps 16 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "reference arm rc=$?"; cut -c1-400 gpurun_out/bench_reference.json
# config 5 (only when its operator is cached on this box: the build takes 10 minutes)
if ls /tmp/h2b_cache/h2b_config5_*/DONE >/dev/null 2>&1; then
timeout 1500 python bench.py --config config5 --steps 10 --warmup 3 > gpurun_out/bench_config5.json 2> gpurun_out/bench_config5.err; echo "config5 rc=$?"; cut -c1-300 gpurun_out/bench_config5.json
timeout 900 python bench.py --config config3 --nrhs 8 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_nrhs8.json 2> gpurun_out/bench_nrhs8.err; echo "nrhs8 rc=$?"
fi
