#!/bin/bash
# Register-cap sweep (DGB_OPTION_MIN_BLOCKS) for configs 2 and 4.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in ${CONFIGS:-2 4}; do for mb in ${MBS:-0 5 6}; do
  python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --minblocks $mb > gpurun_out/mb_c${c}_${mb}.json 2>&1
  f=gpurun_out/mb_c${c}_${mb}.json; python -c "
import json; d=json.load(open('$f')); r=d['roofline']; print('$f', round(d['value']/1e6,1), 'Mel/s', r['kernel_ms'], 'ms', r['achieved'], 'GB/s', r['frac'])" 2>/dev/null || (echo $f; tail -3 $f)
done; done
