#!/bin/bash
# Bench every config, then: launch list (config 2) and full ncu captures of the block-row
# kernel for configs 2, 3 and 4.  Outputs in gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
for c in 1 3 4 5; do
  python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
done
for c in 2 3 4; do
  CMD="python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
  $CMD > gpurun_out/plain_c$c.log 2>&1 || continue
  if [ $c = 2 ]; then
    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches_c2.csv $CMD > gpurun_out/ncu_launch.log 2>&1
  fi
  ncu --set full --clock-control none --import-source on -k regex:assemble_ -s 1 -c 1 \
      -o gpurun_out/prof_c$c $CMD > gpurun_out/ncu_c$c.log 2>&1
done
# summaries on the box (the reports themselves exceed gpurun's 64 MiB return limit)
mkdir -p gpurun_out/prof_new
cp profiles/ncu_summary.json gpurun_out/prof_new/ 2>/dev/null
PROF_DIR=gpurun_out/prof_new python tools/summarize_ncu.py ${TAG:-r01} > gpurun_out/summ.log 2>&1
rm -f gpurun_out/prof_c2.ncu-rep gpurun_out/prof_c3.ncu-rep
ls -la gpurun_out
