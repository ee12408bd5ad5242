#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for mb in 0 3 4; do python bench.py --minblocks $mb --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/tune_c2_mb$mb.json 2>&1; done
for c in 1 3 4; do python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c$c.json 2>&1; done
CMD="python bench.py --config 4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:assemble_kernel -s 1 -c 1 -o gpurun_out/prof_c4 $CMD > gpurun_out/ncu4.log 2>&1
tail -n 2 gpurun_out/ncu4.log
