#!/bin/bash
# Kernel time per config under L2 policies 0 (normal) and 2 (evict-first output).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in ${CONFIGS:-2 3 4 5}; do
  for pol in ${POLS:-0 2}; do
    python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --l2-policy $pol $BENCH_ARGS > gpurun_out/l2_c${c}_p${pol}.json 2>&1
    python -c "
import json; d=json.load(open('gpurun_out/l2_c${c}_p${pol}.json')); r=d['roofline']; print('c$c pol $pol', r['kernel_ms'], 'ms', r['frac'])" 2>/dev/null || tail -3 gpurun_out/l2_c${c}_p${pol}.json
  done
done
