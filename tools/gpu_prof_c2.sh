#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CMD="python bench.py --config 2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:assemble_ -s 1 -c 1 -o gpurun_out/prof_c2 $CMD > gpurun_out/ncu_c2.log 2>&1
tail -2 gpurun_out/ncu_c2.log
