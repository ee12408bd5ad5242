#!/bin/bash
# ncu --set full of config 2's batched kernel (BENCH_ARGS, e.g. --ws 8).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CMD="python bench.py --config 2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline $BENCH_ARGS"
$CMD > gpurun_out/plain_ws.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:assemble_ -s 1 -c 1 -o gpurun_out/prof_ws $CMD > gpurun_out/ncu_ws.log 2>&1
tail -2 gpurun_out/ncu_ws.log
