#!/bin/bash
# Parity suite + short bench lines for configs 2-4 (tuning loop).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | grep -E "passed|failed|Error|assert" | tail -8
for c in ${CONFIGS:-2 3 4}; do
  python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $BENCH_ARGS > gpurun_out/q_c${c}.json 2>&1
done
for c in ${CONFIGS:-2 3 4}; do f=gpurun_out/q_c${c}.json; python -c "
import json; d=json.load(open('$f')); r=d['roofline']; print('$f', round(d['value']/1e6,1), 'Mel/s', r['kernel_ms'], 'ms', r['achieved'], 'GB/s', r['frac'])" 2>/dev/null || (echo $f; tail -3 $f); done
