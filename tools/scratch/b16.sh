#!/bin/bash
mkdir -p gpurun_out
for R in 16 8; do
timeout 900 python bench.py --config config3 --nrhs $R --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_nrhs$R.json 2> gpurun_out/bench_nrhs$R.err; echo "nrhs $R rc=$?"
python - <<P
import json
d=json.loads(open('gpurun_out/bench_nrhs$R.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['roofline']['frac'], d['parity'], d['e2e']['ms_per_step'], [(k['kernel'], k['items'], round(k['ms'],3)) for k in d['roofline']['kernels']])
P
done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
