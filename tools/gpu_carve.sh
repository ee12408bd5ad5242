#!/bin/bash
# Persisting-L2 carve-out x L2 policy sweep on config 4 (kernel ms), with DRAM bytes of one launch.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for pp in ${PP:-1}; do for pol in ${POLS:-2 6}; do for mb in ${MBS:-0}; do
  f=gpurun_out/cv_${pp}_${pol}_${mb}.json
  CMD="python bench.py --config 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --p1-pipe $pp --l2-policy $pol --l2-carve-mb $mb"
  $CMD > $f 2>&1
  python -c "
import json; d=json.load(open('$f')); r=d['roofline']; print('pipe $pp policy $pol carve $mb', r['kernel_ms'], 'ms')" 2>/dev/null || (echo $f; tail -3 $f)
  if [ -n "$DRAM" ]; then
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none \
        -k regex:assemble_ -s 4 -c 1 --csv $CMD 2>/dev/null | grep -E "dram__" | awk -F'","' '{print "   ", $(NF-2), $NF}'
  fi
done; done; done
