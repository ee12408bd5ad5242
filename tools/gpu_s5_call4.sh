#!/bin/bash
set -u
O=gpurun_out
LIB=paper_1502_02941_b200/libdgfem_b200.so
cp abtest/libG6.so $LIB
timeout 900 python -m pytest tests/test_gpu_bench_paths.py tests/test_gpu_parity.py tests/test_gpu_features.py -m gpu -x -q > $O/s5_tests_G6.log 2>&1; echo "rc=$?" >> $O/s5_tests_G6.log
LIBS="F6 G6 G3 G2" REPS=3 tools/gpu_abn.sh > $O/s5_ab4_c4.txt 2>&1
LIBS="F6 G6 G3" REPS=2 OP=c1 tools/gpu_abn.sh > $O/s5_ab4_c1.txt 2>&1
cp abtest/libG6.so $LIB
ncu --set full --import-source on --clock-control none -k regex:assemble_p1_pipe -s 3 -c 1 -o $O/s5_c1b_G6 \
  python bench.py --op c1-throughput --steps 1 --warmup 0 > $O/s5_ncu_c1b.log 2>&1
