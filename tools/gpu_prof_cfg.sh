#!/bin/bash
# ncu --set full of the block-row kernel for one config (CFG env, default 4).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
C=${CFG:-4}
CMD="python bench.py --config $C --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_c$C.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:assemble_ -s 1 -c 1 -o gpurun_out/prof_c$C $CMD > gpurun_out/ncu_c$C.log 2>&1
tail -2 gpurun_out/ncu_c$C.log
