"""Debug aid: config-5 assembly on a small mesh under the ablation switches (one process per
setting, so an illegal access in one does not poison the others)."""
import sys
sys.path.insert(0, '/root/repo')
import torch  # noqa: E402
from paper_1502_02941_b200 import capi, dgfem, problems  # noqa: E402

ab = int(sys.argv[1]) if len(sys.argv) > 1 else 0
cfg = problems.CONFIGS[5]
mesh = dgfem.unit_square_mesh(16, 0.0, 0, False, 0, 0)
ref = dgfem.ReferenceElement(cfg.degree, cfg.quad_order)
spec = problems.config_problem(5, mesh.n_elements)
params = dgfem.config_parameters(cfg, capi.IIPG)
plan = dgfem.Plan(ref.view)
plan.set_option(1000, ab)
dm, dp = dgfem.DeviceMesh(mesh), dgfem.DeviceProblem(spec)
out = plan.assemble(dm, dp, params, plan.allocate(dm), check=False)
torch.cuda.synchronize()
print('ablate', ab, 'ok', flush=True)
