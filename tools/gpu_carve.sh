#!/bin/bash
# Persisting-L2 carve-out sweep on config 4 (kernel ms), one-shot and pipelined P1 kernels.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for pp in ${PP:-0 12}; do for pol in ${POLS:-2 6}; do for mb in ${MBS:-0}; do
  f=gpurun_out/cv_${pp}_${pol}_${mb}.json
  python bench.py --config 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --p1-pipe $pp --l2-policy $pol --l2-carve-mb $mb > $f 2>&1
  python -c "
import json; d=json.load(open('$f')); r=d['roofline']; print('pipe $pp policy $pol carve $mb', r['kernel_ms'], 'ms')" 2>/dev/null || (echo $f; tail -3 $f)
done; done; done
