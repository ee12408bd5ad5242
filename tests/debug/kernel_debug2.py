"""Debug aid: the per-element-fields kernel test body, method by method, with block-level
error attribution."""
import sys
sys.path.insert(0, '/root/repo')
sys.path.insert(0, '/root/repo/tests')
import numpy as np  # noqa: E402
import torch  # noqa: E402
from oracle.oracle import OracleLib  # noqa: E402
from paper_1502_02941_b200 import capi, dgfem, problems  # noqa: E402

deg, qo, vel = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
oracle = OracleLib()
mesh = dgfem.unit_square_mesh(10, 0.2, 31, True, 32, 2)
ref = dgfem.ReferenceElement(deg, qo)
b = {"const": problems.vec_constant(0.8, -0.3),
     "affine": problems.vec_affine(0.5, -0.5, 0.0, -1.0, 1.0, 0.0),
     "trig": problems.vec_trig(2 * problems.PI, 2 * problems.PI)}[vel]
u = (capi.FN_SIN_SIN, (1.0,))
spec = problems.make_problem("kernels", 1.0, b, 1.0, problems.function(*u),
                             problems.function(*u), neumann_sides=2)
r = problems.uniform01(777 + deg, 2 * mesh.n_elements)
spec.set_per_element("diffusion", 10.0 ** (-4.0 + 4.0 * r[:mesh.n_elements]))
spec.set_per_element("linear_reaction", 2.0 * r[mesh.n_elements:])
bound = len(sys.argv) > 4 and sys.argv[4] == "bound"
plan = dgfem.Plan(ref.view)
dm, dp = dgfem.DeviceMesh(mesh), dgfem.DeviceProblem(spec)
if bound:
    plan.bind_mesh(dm)
for method in (capi.SIPG, capi.NIPG, capi.IIPG):
    params = dgfem.set_parameters(method, deg, capi.INFLOW_DROP)
    out = plan.allocate(dm)
    out.val.fill_(float("nan"))
    out.rhs.fill_(float("nan"))
    s = plan.assemble(dm, dp, params, out)
    torch.cuda.synchronize()
    g = (s.row_ptr.cpu().numpy(), s.col.cpu().numpy(), s.val.cpu().numpy(), s.rhs.cpu().numpy())
    o = oracle.assemble(mesh.arrays(), ref.tables(), spec.c, params)
    rp = o[0]
    owner = np.repeat(np.arange(rp.size - 1), np.diff(rp))
    nl = ref.n_local
    scale = np.zeros((rp.size - 1, nl))
    np.maximum.at(scale, owner, np.abs(o[2]).max(axis=2))
    e = np.abs(g[2] - o[2]) / np.maximum(scale[owner][:, :, None], 1e-300)
    bw = e.max(axis=(1, 2))
    w = int(np.argmax(bw))
    nanb = np.argwhere(np.isnan(g[2]))
    print("unwritten entries:", nanb[:10].tolist(), "of", len(nanb), "rhs nan", int(np.isnan(g[3]).sum()))
    print(method, f"max {bw.max():.3e} block {w} row {owner[w]} col {o[1][w]} diag {o[1][w] == owner[w]}",
          "gpu", g[2][w].ravel()[:4], "ref", o[2][w].ravel()[:4], flush=True)
