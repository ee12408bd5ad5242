O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > $O/s4_gputests.log 2>&1; echo "pytest rc=$?" >> $O/s4_gputests.log
python __graft_entry__.py smoke > $O/s4_smoke.log 2>&1; echo "smoke rc=$?" >> $O/s4_smoke.log
python bench.py > $O/s4_bench.json 2> $O/s4_bench.err
python tools/c4_diag.py > $O/s4_diag.log 2>&1
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --secondary ''"
eval ncu --set full --clock-control none --import-source on -k regex:assemble_p1_pipe -s 2 -c 1 -o $O/s4_c4 $B > $O/s4_ncu_c4.log 2>&1
ls -la $O
