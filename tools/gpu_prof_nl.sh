#!/bin/bash
# ncu --set full of the nonlinear-reaction kernel (bench.py --op nonlinear, config CFG).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
C=${CFG:-2}
CMD="python bench.py --op nonlinear --config $C --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_nl.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:nonlinear_kernel -s 1 -c 1 -o gpurun_out/prof_nl_c$C $CMD > gpurun_out/ncu_nl.log 2>&1
tail -2 gpurun_out/ncu_nl.log
