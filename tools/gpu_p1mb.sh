#!/bin/bash
# P1 kernel variants on config 4: register budget (--minblocks 4/5/6) after a parity run.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | grep -E "passed|failed|Error|assert" | tail -8
for mb in ${MBS:-0 5 6}; do
  f=gpurun_out/mb_c4_$mb.json
  python bench.py --config 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --minblocks $mb > $f 2>&1
  python -c "
import json; d=json.load(open('$f')); r=d['roofline']; print('c4 minblocks $mb', r['kernel_ms'], 'ms', r['frac'])" 2>/dev/null || (echo $f; tail -3 $f)
done
