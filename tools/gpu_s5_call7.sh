#!/bin/bash
set -u
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > $O/s5_gputests.log 2>&1; echo "pytest rc=$?" >> $O/s5_gputests.log
python __graft_entry__.py smoke > $O/s5_smoke.log 2>&1; echo "smoke rc=$?" >> $O/s5_smoke.log
python bench.py > $O/s5_bench.json 2> $O/s5_bench.err
python bench.py --op c1-throughput > $O/s5_c1.json 2> $O/s5_c1.err
python bench.py --op c1-throughput --copies 4096 > $O/s5_c1_4096.json 2> $O/s5_c1_4096.err
