#!/bin/bash
# ncu evidence for the bench (run on the GPU box via gpurun).
#  1) launch list of the bench command (cold, serialised: compare SHARES)
#  2) one --set full capture of the persistent executor kernel
set -x
OUT=${1:-gpurun_out}
mkdir -p $OUT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > $OUT/ncu_bench_stdout.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:serinv_exec -s 1 -c 1 \
  -o $OUT/prof_exec python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > $OUT/ncu_full_stdout.txt 2>&1
ls -la $OUT
