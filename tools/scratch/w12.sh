#!/bin/bash
mkdir -p gpurun_out
G='{}'
timeout 900 python tools/sweep.py --config config3 --steps 20 --grid "$G" --nrhs 8,16 > gpurun_out/t384_c3.jsonl 2> gpurun_out/t384_c3.err; echo "default (384) rc=$?"; cut -c1-150 gpurun_out/t384_c3.jsonl
for T in 448 512; do
H2B_LIB=$PWD/paper_1811_05731_b200/libh2b_t$T.so timeout 900 python tools/sweep.py --config config3 --steps 20 --grid "$G" --nrhs 8,16 > gpurun_out/t${T}_c3.jsonl 2> gpurun_out/t${T}_c3.err; echo "t$T rc=$?"; cut -c1-150 gpurun_out/t${T}_c3.jsonl; tail -2 gpurun_out/t${T}_c3.err | cut -c1-200
done
