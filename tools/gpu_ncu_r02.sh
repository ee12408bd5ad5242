#!/bin/bash
# Round-2 ncu evidence (1 GPU; every ncu run preceded by the same command run plain, exit 0).
# PART a: tests, mesh, config-1 throughput, launch list, C4 capture; b: SpMV, C2, C3; c: C5
# (split so each call's gpurun_out/ stays under 64 MiB)
O=gpurun_out
P=${1:-a}
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --secondary ''"
if [ "$P" = a ]; then
  timeout 600 python -m pytest tests/test_gpu_device_mesh.py tests/test_gpu_bench_paths.py -q > $O/n2_tests.log 2>&1
  python bench.py --op mesh > $O/n2_mesh_a.json 2>&1; python bench.py --op mesh > $O/n2_mesh_b.json 2>&1
  python bench.py --op c1-throughput > $O/n2_c1tp.json 2>&1
  eval $B > $O/n2_plain_c4.log 2>&1 && \
    eval ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_r02_c4.csv $B > $O/n2_ncu_launch.log 2>&1
  eval $B > $O/n2_plain_c4b.log 2>&1 && \
    eval ncu --set full --clock-control none --import-source on -k regex:assemble_p1_pipe -s 2 -c 1 -o $O/r02_c4 $B > $O/n2_ncu_c4.log 2>&1
fi
if [ "$P" = b ]; then
  S="python bench.py --op spmv --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
  $S > $O/n2_plain_spmv.log 2>&1 && \
    ncu --set full --clock-control none -k regex:bsr_spmv -s 3 -c 1 -o $O/r02_spmv $S > $O/n2_ncu_spmv.log 2>&1
  C2="python bench.py --config 2 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --secondary ''"
  eval $C2 > $O/n2_plain_c2.log 2>&1 && \
    eval ncu --set full --clock-control none -k regex:assemble_ws -s 2 -c 1 -o $O/r02_c2 $C2 > $O/n2_ncu_c2.log 2>&1
  C3="python bench.py --config 3 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --secondary ''"
  eval $C3 > $O/n2_plain_c3.log 2>&1 && \
    eval ncu --set full --clock-control none -k regex:assemble_kernel -s 2 -c 1 -o $O/r02_c3 $C3 > $O/n2_ncu_c3.log 2>&1
fi
if [ "$P" = c ]; then
  C5="python bench.py --config 5 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --secondary ''"
  eval $C5 > $O/n2_plain_c5.log 2>&1 && \
    eval ncu --set full --clock-control none --import-source on -k regex:assemble_kernel -s 2 -c 1 -o $O/r02_c5 $C5 > $O/n2_ncu_c5.log 2>&1
fi
