#!/bin/bash
# Session-5 call 1: variants of the persistent P1 kernel (A = HEAD, B = extended geometry record +
# chunk tickets, C = extended record with static chunks), per-warp diagnostics (D, tuning build)
set -u
O=gpurun_out
LIB=paper_1502_02941_b200/libdgfem_b200.so
cp abtest/libB.so $LIB
timeout 900 python -m pytest tests/test_gpu_bench_paths.py tests/test_gpu_parity.py tests/test_gpu_features.py -m gpu -x -q > $O/s5_tests_B.log 2>&1; echo "rc=$?" >> $O/s5_tests_B.log
LIBS="A B C" REPS=3 tools/gpu_abn.sh > $O/s5_ab_c4.txt 2>&1
LIBS="A B C" REPS=2 OP=c1 tools/gpu_abn.sh > $O/s5_ab_c1.txt 2>&1
cp abtest/libD.so $LIB
python tools/p1_diag.py > $O/s5_diag.txt 2>&1
cp abtest/libB.so $LIB
ncu --set full --import-source on --clock-control none -k regex:assemble_p1_pipe -c 1 -o $O/s5_c4_B \
  python bench.py --config 4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/s5_ncu.log 2>&1
