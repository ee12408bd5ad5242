#!/bin/bash
# L2 policy x ablation grid for one config (CFG), kernel ms only.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for pol in ${POLS:-2 6 4}; do for ab in ${ABL:-0 32}; do
  f=gpurun_out/la_${pol}_${ab}.json
  python bench.py --config ${CFG:-4} --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --l2-policy $pol --ablate $ab > $f 2>&1
  python -c "
import json; d=json.load(open('$f')); r=d['roofline']; print('policy $pol ablate $ab', r['kernel_ms'], 'ms')" 2>/dev/null || (echo $f; tail -3 $f)
done; done
