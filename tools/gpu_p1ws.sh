#!/bin/bash
# P1 on the warp-specialised tensor-core kernel (option --ws n) vs the P1 kernel (--ws 0).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | grep -E "passed|failed|Error|assert" | tail -8
for c in ${CONFIGS:-4}; do for w in ${WS:-0 8 10 12}; do
  f=gpurun_out/pw_c${c}_$w.json
  python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --ws $w > $f 2>&1
  python -c "
import json; d=json.load(open('$f')); r=d['roofline']; print('c$c ws $w', r['kernel_ms'], 'ms', r['frac'])" 2>/dev/null || (echo $f; tail -3 $f)
done; done
