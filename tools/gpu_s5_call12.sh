#!/bin/bash
set -u
O=gpurun_out
LIB=paper_1502_02941_b200/libdgfem_b200.so
cp abtest/libJ1.so $LIB
timeout 900 python -m pytest tests/test_gpu_bench_paths.py tests/test_gpu_parity.py tests/test_gpu_features.py -m gpu -x -q > $O/s5_tests_J1.log 2>&1; echo "rc=$?" >> $O/s5_tests_J1.log
LIBS="K J0 J1" REPS=3 tools/gpu_abn.sh > $O/s5_ab12_c4.txt 2>&1
LIBS="K J0 J1" REPS=2 OP=c1 tools/gpu_abn.sh > $O/s5_ab12_c1.txt 2>&1
