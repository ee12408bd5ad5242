"""Debug aid: does one entry depend on the output buffer's previous content?"""
import sys
sys.path.insert(0, '/root/repo')
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1502_02941_b200 import capi, dgfem, problems  # noqa: E402

deg, qo = 1, 3
mesh = dgfem.unit_square_mesh(10, 0.2, 31, True, 32, 2)
ref = dgfem.ReferenceElement(deg, qo)
b = problems.vec_affine(0.5, -0.5, 0.0, -1.0, 1.0, 0.0)
u = (capi.FN_SIN_SIN, (1.0,))
spec = problems.make_problem("k", 1.0, b, 1.0, problems.function(*u), problems.function(*u), neumann_sides=2)
r = problems.uniform01(778, 2 * mesh.n_elements)
spec.set_per_element("diffusion", 10.0 ** (-4.0 + 4.0 * r[:mesh.n_elements]))
spec.set_per_element("linear_reaction", 2.0 * r[mesh.n_elements:])
plan = dgfem.Plan(ref.view)
dm, dp = dgfem.DeviceMesh(mesh), dgfem.DeviceProblem(spec)
params = dgfem.set_parameters(capi.SIPG, deg, capi.INFLOW_DROP)
for fill in (None, 0.0, float("nan"), 7.0, None):
    out = plan.allocate(dm)
    if fill is not None:
        out.val.fill_(fill)
    torch.cuda.synchronize()
    plan.assemble(dm, dp, params, out)
    torch.cuda.synchronize()
    v = out.val.cpu().numpy()
    print("fill", fill, "entry", v[757, 0, 0], "row 198 last", v[756].ravel()[-1], "block 759 last", v[759].ravel()[-1], flush=True)
