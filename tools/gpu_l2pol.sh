#!/bin/bash
# L2 policy sweep (plan option L2_POLICY) for one config.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for pol in 0 1 2 3; do
  python bench.py --config ${CFG:-4} --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --l2-policy $pol > gpurun_out/l2_$pol.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/l2_$pol.json')); r=d['roofline']; print('policy $pol', r['kernel_ms'], 'ms', r['frac'])" 2>/dev/null || tail -3 gpurun_out/l2_$pol.json
done
