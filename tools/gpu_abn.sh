#!/bin/bash
# Same-box A/B/... of library builds abtest/lib<X>.so (LIBS="A B C"): alternating bench runs of
# one config (CFG, default 4; OP=c1 times the 512-system config-1 batch instead).
cd "$(dirname "$0")/.."
LIB=paper_1502_02941_b200/libdgfem_b200.so
cp $LIB /tmp/lib_cur.so
for i in $(seq 1 ${REPS:-3}); do for v in ${LIBS:-A B}; do
  cp abtest/lib$v.so $LIB
  if [ "${OP:-}" = c1 ]; then
    python bench.py --op c1-throughput --steps 20 --warmup 5 $BENCH_ARGS | \
      python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('$v c1-batch', r.get('kernel_ms'), r.get('frac'))"
  else
    python bench.py --config ${CFG:-4} --steps 20 --warmup 5 --no-e2e --no-cpu-baseline $BENCH_ARGS | \
      python -c "import json,sys; d=json.load(sys.stdin)['roofline']; print('$v', d['kernel_ms'], d['frac'])"
  fi
done; done
cp /tmp/lib_cur.so $LIB
