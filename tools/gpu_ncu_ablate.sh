#!/bin/bash
cd /root/repo
for ab in 16 0; do
python bench.py --config 2 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --ablate $ab > gpurun_out/abn_$ab.json 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,smsp__cycles_active.avg --clock-control none -k regex:assemble_ -c 6 --csv python bench.py --config 2 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --ablate $ab 2>/dev/null | grep -E "gpu__time|cycles_active" | head -9
done
