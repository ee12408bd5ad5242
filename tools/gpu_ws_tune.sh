#!/bin/bash
# Producer-warp count of the warp-specialised kernel (0 = monolithic), config 2, batched and not.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for extra in "" "--no-batch"; do
  for ws in ${WS:-0 4 6 8 10 12}; do
    python bench.py --config 2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --ws $ws $extra > gpurun_out/ws.json 2>&1
    python -c "
import json; d=json.load(open('gpurun_out/ws.json')); r=d['roofline']; print('ws $ws $extra', r['kernel_ms'], 'ms', r['frac'])" 2>/dev/null || tail -3 gpurun_out/ws.json
  done
done
