"""Iterations and wall time of dgb_solve on configs 1 and 2 (restart lengths 30/60)."""
import sys
import time

sys.path.insert(0, '/root/repo')
import torch  # noqa: E402

from paper_1502_02941_b200 import capi, dgfem, problems  # noqa: E402

for c in (1, 2):
    cfg = problems.CONFIGS[c]
    mesh = dgfem.config_mesh(cfg)
    spec = problems.config_problem(c, mesh.n_elements)
    ref = dgfem.ReferenceElement(cfg.degree, cfg.quad_order)
    plan = dgfem.Plan(ref.view)
    dm, dp = dgfem.DeviceMesh(mesh), dgfem.DeviceProblem(spec)
    out = plan.assemble(dm, dp, dgfem.config_parameters(cfg, capi.SIPG), plan.allocate(dm))
    for m in (30, 60):
        for rep in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            x, info = dgfem.solve(out, out.rhs.reshape(-1), options=dgfem.solve_options(restart=m))
            torch.cuda.synchronize()
            t = time.perf_counter() - t0
        print(c, m, 'its', info['iterations'], 'time %.4f s' % t, 'us/it %.1f' % (1e6 * t / info['iterations']),
              'defect', info['defect_norm2'], info['bound'], flush=True)
