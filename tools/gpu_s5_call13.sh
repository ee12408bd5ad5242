#!/bin/bash
set -u
O=gpurun_out
LIB=paper_1502_02941_b200/libdgfem_b200.so
timeout 900 python -m pytest tests/test_gpu_bench_paths.py tests/test_gpu_parity.py tests/test_gpu_features.py -m gpu -q > $O/s5_tests_L.log 2>&1; echo "rc=$?" >> $O/s5_tests_L.log
LIBS="K L" REPS=3 tools/gpu_abn.sh > $O/s5_ab13_c4.txt 2>&1
LIBS="K L" REPS=2 OP=c1 tools/gpu_abn.sh > $O/s5_ab13_c1.txt 2>&1
