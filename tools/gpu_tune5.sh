#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in 2 4 3; do for l2 in 0 1 2 3; do
  python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --l2-policy $l2 > gpurun_out/tune_c${c}_l2$l2.json 2>&1
done; done
for f in gpurun_out/tune_c*_l2*.json; do python -c "
import json; d=json.load(open('$f')); r=d['roofline']; print('$f', round(d['value']/1e6,1), 'Mel/s', r['kernel_ms'], 'ms', r['achieved'], 'GB/s', r['frac'])" 2>/dev/null || (echo $f; tail -3 $f); done
