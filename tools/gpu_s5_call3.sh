#!/bin/bash
set -u
O=gpurun_out
LIB=paper_1502_02941_b200/libdgfem_b200.so
cp abtest/libF6.so $LIB
timeout 900 python -m pytest tests/test_gpu_bench_paths.py tests/test_gpu_parity.py tests/test_gpu_features.py -m gpu -x -q > $O/s5_tests_F6.log 2>&1; echo "rc=$?" >> $O/s5_tests_F6.log
LIBS="E1 F6 F3 F2" REPS=2 OP=c1 tools/gpu_abn.sh > $O/s5_ab3_c1.txt 2>&1
LIBS="F6" REPS=1 OP=c1 BENCH_ARGS="--copies 4096" tools/gpu_abn.sh >> $O/s5_ab3_c1.txt 2>&1
cp abtest/libF6.so $LIB
ncu --set full --import-source on --clock-control none -k regex:assemble_p1_pipe -c 1 -o $O/s5_c4_F6 \
  python bench.py --config 4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/s5_ncu_F6.log 2>&1
