"""Same-process A/B of the P1 persistent kernel with and without the bound vertex coordinates
(DGB_OPTION_GEOMETRY_CACHE) on config 4 and the 512-system config-1 batch; outputs compared
bitwise (tools only)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1502_02941_b200 import capi, workload  # noqa: E402

stream = torch.cuda.current_stream()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for cfg in (4, 1):
    ref = None
    for v in (1, 0, 1, 0):
        if cfg == 1:
            run = workload.BatchedSystemsRun(1, 512, options={capi.OPTION_GEOMETRY_CACHE: v})
        else:
            run = workload.ConfigRun(cfg, options={capi.OPTION_GEOMETRY_CACHE: v})
        s_ms, k_ms = bench.time_steps(run, stream, 20, 5, flush)
        d = bench.device_summary(run, s_ms, k_ms)
        out = run.outputs()[0]
        cur = (out.val, out.rhs, out.col, out.row_ptr)
        if ref is None:
            ref = tuple(t.clone() for t in cur)
            diff = "reference"
        else:
            diff = "bitwise equal: " + str(all(torch.equal(a, b) for a, b in zip(cur, ref)))
        print(f"config {cfg} geometry cache {v}: kernel {d['kernel_ms']:.4f} ms  frac {d['frac']:.4f}  bind {run.bind_ms:.2f} ms  {diff}", flush=True)
        del run, out, cur
        torch.cuda.empty_cache()
