#!/bin/bash
set -u
O=gpurun_out
LIB=paper_1502_02941_b200/libdgfem_b200.so
cp abtest/libI6.so $LIB
timeout 900 python -m pytest tests/test_gpu_bench_paths.py tests/test_gpu_parity.py tests/test_gpu_features.py -m gpu -q > $O/s5_tests_I6.log 2>&1; echo "rc=$?" >> $O/s5_tests_I6.log
LIBS="E1 H6 I6 I3 I6e" REPS=3 tools/gpu_abn.sh > $O/s5_ab6_c4.txt 2>&1
LIBS="H6 I6 I3 I6e" REPS=2 OP=c1 tools/gpu_abn.sh > $O/s5_ab6_c1.txt 2>&1
