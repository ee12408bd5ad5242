#!/bin/bash
# Time attribution for the P2 kernel (results wrong while ablating): see dgb_plan_set_option 1000.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in ${CONFIGS:-2}; do for ab in ${ABL:-0 1 2 4 8 12 13 15}; do
  python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --ablate $ab > gpurun_out/ab_c${c}_${ab}.json 2>&1
  f=gpurun_out/ab_c${c}_${ab}.json; python -c "
import json; d=json.load(open('$f')); r=d['roofline']; print('$f', r['kernel_ms'], 'ms')" 2>/dev/null || (echo $f; tail -3 $f)
done; done
