#!/bin/bash
# config 5 with the GPU recompression (default): build log, memory guard, bench with the operator check, structure vs fixture
mkdir -p gpurun_out
MEMGUARD_MIN_KB=12000000 tools/memguard.sh gpurun_out/c5rc_guard.log python bench.py --config config5 --steps 10 --warmup 3 > gpurun_out/c5rc_bench.json 2> gpurun_out/c5rc_bench.err; echo "bench rc=$?"
tail -2 gpurun_out/c5rc_guard.log
grep -i "recompress\|operator check\|parity\|HCA (gpu): [0-9]* blocks,\|near field\|surface" gpurun_out/c5rc_bench.err | cut -c1-420
python - <<'P'
import json, numpy as np
d=json.loads(open('gpurun_out/c5rc_bench.json').read().strip().splitlines()[-1])
print('ms', d['ms_per_step'], 'h2_bytes', d['config']['h2_bytes'], 'fixture', int(np.load('tests/golden/config5_structure.npz')['storage_bytes']))
print(d['operator_check'])
print(d['build']['seconds'])
P
