#!/bin/bash
set -u
O=gpurun_out
python tools/c1_batch_once.py > $O/s5_c1once.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:assemble_p1_pipe -s 2 -c 1 -o $O/s5_c1batch python tools/c1_batch_once.py > $O/s5_ncu_c1batch.log 2>&1
