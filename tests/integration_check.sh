#!/bin/bash
# Builds the INTEGRATION.md adapter (include/dgfem/gpu.hpp, extracted from the doc) against the
# unmodified reference objects in oracle/_ref/obj and runs assemble_all through it, comparing
# the GPU result with the reference's own stiffness()/F.  Needs oracle/_ref (built in the
# container that has /root/reference; the objects travel with the repo snapshot).
set -e
cd "$(dirname "$0")/.."
OUT=gpurun_out/integration
mkdir -p $OUT/dgfem
python - <<'PY'
import re
s = open("INTEGRATION.md").read()
code = re.search(r"```cpp\n(// include/dgfem/gpu.hpp.*?)```", s, re.S).group(1)
open("gpurun_out/integration/dgfem/gpu.hpp", "w").write(code)
PY
REFINC=oracle/_ref/include
[ -d /root/reference/proj/include ] && REFINC=/root/reference/proj/include
g++ -std=c++20 -O2 -I$OUT -I$REFINC -Iinclude tests/integration/main.cpp oracle/_ref/obj/*.o \
    paper_1502_02941_b200/libdgfem_b200.so -fopenmp -o $OUT/integ
LD_LIBRARY_PATH=paper_1502_02941_b200 $OUT/integ
