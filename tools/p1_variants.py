"""Times the P1 block-row kernel variants (DGB_OPTION_P1_PIPELINE 1: persistent pipelined,
0: one-shot) on config 4 (or config 1 batched) and checks each against the first one's output
(tools only; tools/experiments/assemble_p1_tri.cuh was measured this way, see
profiles/NOTES.md)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1502_02941_b200 import capi, workload  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
variants = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 0]
stream = torch.cuda.current_stream()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
ref = None
for v in variants:
    if cfg == 1:
        run = workload.BatchedSystemsRun(1, 512)
        run.plan.set_option(capi.OPTION_P1_PIPELINE, v)
    else:
        run = workload.ConfigRun(cfg, options={capi.OPTION_P1_PIPELINE: v})
    s_ms, k_ms = bench.time_steps(run, stream, 20, 3, flush)
    d = bench.device_summary(run, s_ms, k_ms)
    out = run.outputs()[0]
    if ref is None:
        ref = (out.val.clone(), out.rhs.clone(), out.col.clone(), out.row_ptr.clone())
        diff = "reference"
    else:
        dv = ((out.val - ref[0]).abs().max() / ref[0].abs().max()).item()
        dr = ((out.rhs - ref[1]).abs().max() / ref[1].abs().max()).item()
        pat = torch.equal(out.col, ref[2]) and torch.equal(out.row_ptr, ref[3])
        diff = f"max|dK|/max|K| {dv:.2e}  max|dF|/max|F| {dr:.2e}  pattern equal {pat}"
    print(f"p1 variant {v}: kernel {d['kernel_ms']:.4f} ms  frac {d['frac']:.4f}  {diff}", flush=True)
    del run
    torch.cuda.empty_cache()
