#!/bin/bash
# gpu_quick.sh, then one ncu --set full capture of the config-2 kernel.
cd "$(dirname "$0")/.."
bash tools/gpu_quick.sh
rm -f gpurun_out/prof_c2.ncu-rep
bash tools/gpu_prof_c2.sh
