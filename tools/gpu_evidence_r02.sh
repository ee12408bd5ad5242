#!/bin/bash
# Round-2 evidence run (1 GPU): GPU suite, smoke, every bench op, reference arm -> gpurun_out/
set -u
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv > $O/e2_smi.txt
timeout 1500 python -m pytest tests -m gpu -q > $O/e2_gputests.log 2>&1; echo "pytest rc=$?" >> $O/e2_gputests.log
python __graft_entry__.py smoke > $O/e2_smoke.log 2>&1; echo "smoke rc=$?" >> $O/e2_smoke.log
python bench.py > $O/e2_bench.json 2> $O/e2_bench.err
python bench.py --impl reference > $O/e2_reference.json 2> $O/e2_reference.err
python bench.py --op spmv > $O/e2_spmv.json 2> $O/e2_spmv.err
python bench.py --op c1-throughput > $O/e2_c1tp.json 2> $O/e2_c1tp.err
python bench.py --op nonlinear --config 4 > $O/e2_nl4.json 2> $O/e2_nl4.err
python bench.py --op solve --config 1 > $O/e2_solve1.json 2> $O/e2_solve1.err
python bench.py --op mesh > $O/e2_mesh_a.json 2> $O/e2_mesh_a.err
python bench.py --op mesh > $O/e2_mesh_b.json 2> $O/e2_mesh_b.err
for c in 2 3 5 1; do python bench.py --config $c > $O/e2_c$c.json 2> $O/e2_c$c.err; done
