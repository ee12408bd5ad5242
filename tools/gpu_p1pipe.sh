#!/bin/bash
# P1 pipelined kernel: parity suite, then config 4 (and 1) per warp count.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | grep -E "passed|failed|Error|assert" | tail -8
for c in ${CONFIGS:-4 1}; do for w in ${WS:-0 1 8 9}; do
  f=gpurun_out/pp_c${c}_$w.json
  python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --p1-pipe $w $BENCH_ARGS > $f 2>&1
  python -c "
import json; d=json.load(open('$f')); r=d['roofline']; print('c$c pipe $w', r['kernel_ms'], 'ms', r['frac'])" 2>/dev/null || (echo $f; tail -3 $f)
done; done
