#!/bin/bash
# One gpurun call: bench every config, then an ncu launch list and a full capture of the
# block-row kernel on the default (config 2) workload.  Outputs land in gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
for c in 1 3 4 5; do
  python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
done
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/launches_c2.csv $CMD > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:assemble_ -s 3 -c 1 \
    -o gpurun_out/prof_c2 $CMD > gpurun_out/ncu2.log 2>&1
for f in gpurun_out/*.err gpurun_out/ncu*.log; do echo "== $f"; tail -n 3 "$f"; done
