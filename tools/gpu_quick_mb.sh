#!/bin/bash
# gpu_quick.sh then the register-cap sweep.
cd "$(dirname "$0")/.."
bash tools/gpu_quick.sh
bash tools/gpu_tune_mb.sh
