"""Config-4 diagnostics: the bound P1 kernel on the config's permuted numbering against the same
2048^2 mesh in structured numbering (what the gather locality costs), tools only."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1502_02941_b200 import dgfem, problems, workload  # noqa: E402

stream = torch.cuda.current_stream()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
cfg = problems.CONFIGS[4]
for name, mesh in (("permuted (config 4)", None), ("structured numbering", dgfem.unit_square_mesh(cfg.n))):
    run = workload.ConfigRun(4, mesh=mesh)
    for rep in range(2):
        s_ms, k_ms = bench.time_steps(run, stream, 20, 3, flush)
        d = bench.device_summary(run, s_ms, k_ms)
        print(f"{name}: kernel {d['kernel_ms']:.4f} ms  frac {d['frac']:.4f}", flush=True)
    del run
    torch.cuda.empty_cache()
