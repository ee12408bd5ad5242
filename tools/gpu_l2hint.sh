#!/bin/bash
# C4 load-hint sweep: bench lines plus steady-state DRAM bytes of one launch (warm caches).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for pol in ${POLS:-2 6 7 3}; do
  CMD="python bench.py --config ${CFG:-4} --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --l2-policy $pol"
  $CMD > gpurun_out/l2h_$pol.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/l2h_$pol.json')); r=d['roofline']; print('policy $pol', r['kernel_ms'], 'ms', r['frac'])" 2>/dev/null || tail -3 gpurun_out/l2h_$pol.json
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --cache-control none --clock-control none \
      -k regex:assemble_ -s 4 -c 1 --csv $CMD 2>/dev/null | grep -E "dram__|gpu__time|lts__" | awk -F'","' '{print "   ", $(NF-2), $NF}'
done
