import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_1502_02941_b200 import capi, dgfem, problems
for c in (1, 2, 4):
    cfg = problems.CONFIGS[c]
    mesh = dgfem.config_mesh(cfg)
    spec = problems.config_problem(c, mesh.n_elements)
    ref = dgfem.ReferenceElement(cfg.degree, cfg.quad_order)
    plan = dgfem.Plan(ref.view)
    dm, dp = dgfem.DeviceMesh(mesh), dgfem.DeviceProblem(spec)
    out = plan.assemble(dm, dp, dgfem.config_parameters(cfg, capi.SIPG), plan.allocate(dm))
    for m in (30, 60, 120):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        try:
            x, info = dgfem.solve(out, out.rhs.reshape(-1), options=dgfem.solve_options(restart=m, max_iterations=20000))
            torch.cuda.synchronize(); t = time.perf_counter() - t0
            print(c, m, 'its', info['iterations'], 'restarts', info['restarts'], 'time %.3f s' % t, 'defect', info['defect_norm2'], info['bound'], flush=True)
        except Exception as e:
            print(c, m, 'ERR', e, time.perf_counter() - t0, flush=True)
