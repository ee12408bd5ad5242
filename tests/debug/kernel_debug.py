"""Debug aid: where a kernel differs from the oracle (block kind, boundary vs interior),
toggling per-element fields and the Neumann side.  python tests/debug/kernel_debug.py DEG QO VEL"""
import sys
sys.path.insert(0, '/root/repo')
sys.path.insert(0, '/root/repo/tests')
import numpy as np  # noqa: E402
import torch  # noqa: E402
from oracle.oracle import OracleLib  # noqa: E402
from paper_1502_02941_b200 import capi, dgfem, problems  # noqa: E402

deg, qo, vel = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
orc = OracleLib()
for per_el in (False, True):
    for sides in (0, 2):
        mesh = dgfem.unit_square_mesh(10, 0.2, 31, True, 32, sides)
        ref = dgfem.ReferenceElement(deg, qo)
        b = {"const": problems.vec_constant(0.8, -0.3),
             "affine": problems.vec_affine(0.5, -0.5, 0.0, -1.0, 1.0, 0.0),
             "trig": problems.vec_trig(2 * problems.PI, 2 * problems.PI)}[vel]
        u = (capi.FN_SIN_SIN, (1.0,))
        spec = problems.make_problem("k", 1.0, b, 1.0, problems.function(*u), problems.function(*u),
                                     neumann_sides=sides)
        if per_el:
            r = problems.uniform01(777 + deg, 2 * mesh.n_elements)
            spec.set_per_element("diffusion", 10.0 ** (-4.0 + 4.0 * r[:mesh.n_elements]))
            spec.set_per_element("linear_reaction", 2.0 * r[mesh.n_elements:])
        method = int(sys.argv[4]) if len(sys.argv) > 4 else capi.SIPG
        params = dgfem.set_parameters(method, deg, capi.INFLOW_DROP)
        s = dgfem.assemble_all(mesh, ref, spec, params)
        torch.cuda.synchronize()
        g = (s.row_ptr.cpu().numpy(), s.col.cpu().numpy(), s.val.cpu().numpy(), s.rhs.cpu().numpy())
        o = orc.assemble(mesh.arrays(), ref.tables(), spec.c, params)
        rp = o[0]
        err = np.abs(g[2] - o[2]).max(axis=(1, 2)) / np.maximum(np.abs(o[2]).max(axis=(1, 2)), 1e-300)
        owner = np.repeat(np.arange(rp.size - 1), np.diff(rp))
        diag = o[1] == owner
        ferr = (np.abs(g[3] - o[3]).max(axis=1) / np.maximum(np.abs(o[3]).max(axis=1), 1e-300)).max()
        worst = int(np.argmax(err))
        print(f"per_el={per_el} sides={sides}: K err diag {err[diag].max():.2e} off {err[~diag].max() if (~diag).any() else 0:.2e}"
              f" F {ferr:.2e}; worst block {worst} row {owner[worst]} col {o[1][worst]} nb {np.diff(rp)[owner[worst]]}", flush=True)
