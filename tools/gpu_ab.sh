#!/bin/bash
# Same-box A/B of two builds of the library (abtest/libA.so, abtest/libB.so): alternating
# bench runs of one config (CFG, default 4).
cd "$(dirname "$0")/.."
LIB=paper_1502_02941_b200/libdgfem_b200.so
cp $LIB /tmp/lib_cur.so
for i in 1 2 3; do for v in A B; do
  cp abtest/lib$v.so $LIB
  python bench.py --config ${CFG:-4} --steps 20 --warmup 5 --no-e2e --no-cpu-baseline $BENCH_ARGS | \
    python -c "import json,sys; d=json.load(sys.stdin)['roofline']; print('$v', d['kernel_ms'], d['frac'])"
done; done
cp /tmp/lib_cur.so $LIB
