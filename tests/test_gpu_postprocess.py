"""GPU: dgb_l2_error / dgb_project / dgb_eval_solution (postprocess.cpp:14-93) against the
C restatement pinned to the reference, and the closed config-1 loop on the device: assemble,
solve, L2 error against the exact solution.  SURVEY.md §8(f) ranks 2 and 4."""
import os

import numpy as np
import pytest

from oracle import newton as onewton
from oracle.oracle import OracleLib, bsr_to_csr
from paper_1502_02941_b200 import capi, dgfem, problems

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "postprocess.npz")


@pytest.fixture(scope="module")
def orc():
    return OracleLib()


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_postprocess_matches_reference_golden(k):
    import torch
    z = np.load(GOLDEN)
    m = dgfem.build_mesh(z["in_nodes"], z["in_elements"], z["in_dirichlet"], z["in_neumann"])
    dm = dgfem.DeviceMesh(m)
    ref = dgfem.ReferenceElement(k)
    coef = torch.from_numpy(z[f"k{k}/coef"]).cuda()
    err, h = dgfem.l2_error(coef, dm, ref, problems.function(capi.FN_SIN_SIN, (1.0,)))
    e_ref, h_ref = z[f"k{k}/l2"]
    assert abs(err - e_ref) <= 1e-12 * e_ref
    assert abs(h - h_ref) <= 2.3e-16 * h_ref       # hypot: correctly rounded here, glibc's is not
    pr = dgfem.project(dm, ref, problems.function(capi.FN_GAUSSIAN, (50.0, 0.5, 0.5))).cpu().numpy()
    pz = z[f"k{k}/project"].reshape(-1, ref.n_local)
    scale = np.maximum(np.abs(pz).max(axis=1, keepdims=True), 1e-300)
    assert (np.abs(pr.reshape(pz.shape) - pz) / scale).max() <= 1e-12
    el = torch.from_numpy(z[f"k{k}/el"]).cuda()
    v = dgfem.eval_solution(coef, ref, el, torch.from_numpy(z[f"k{k}/xh"]).cuda(),
                            torch.from_numpy(z[f"k{k}/yh"]).cuda()).cpu().numpy()
    cz = z[f"k{k}/coef"].reshape(-1, ref.n_local)
    vscale = np.abs(cz[z[f"k{k}/el"]]).sum(axis=1) * 10.0  # |basis| <= ~10 on the triangle
    assert np.all(np.abs(v - z[f"k{k}/eval"]) <= 1e-12 * vscale)


def test_eval_rejects_bad_element():
    import torch
    ref = dgfem.ReferenceElement(1)
    coef = torch.zeros(3 * 8, dtype=torch.float64, device="cuda")
    el = torch.tensor([0, 3, 8, 2], dtype=torch.int32, device="cuda")
    x = torch.zeros(4, dtype=torch.float64, device="cuda")
    with pytest.raises(dgfem.Error) as e:
        dgfem.eval_solution(coef, ref, el, x, x)
    assert e.value.code == "InvalidIndex" and e.value.detail == 2


def test_l2_length_mismatch():
    import torch
    m = dgfem.unit_square_mesh(4)
    with pytest.raises(dgfem.Error) as e:
        dgfem.l2_error(torch.zeros(5, dtype=torch.float64, device="cuda"), dgfem.DeviceMesh(m),
                       dgfem.ReferenceElement(1), problems.function(capi.FN_SIN_SIN, (1.0,)))
    assert e.value.code == "DimensionMismatch"


def test_config1_closed_loop(orc):
    """Config 1 on the device end to end: assemble (SIPG), solve, L2 error against the exact
    solution sin(pi x) sin(pi y).  The same chain on the CPU (restated reference: oracle
    assembly, SuperLU solve, oracle l2_error) agrees to 1e-8 relative."""
    cfg = problems.CONFIGS[1]
    mesh = dgfem.config_mesh(cfg)
    spec = problems.config_problem(1)
    ref = dgfem.ReferenceElement(cfg.degree, cfg.quad_order)
    plan = dgfem.Plan(ref.view)
    dm, dp = dgfem.DeviceMesh(mesh), dgfem.DeviceProblem(spec)
    p = dgfem.config_parameters(cfg, capi.SIPG)
    out = plan.assemble(dm, dp, p, plan.allocate(dm))
    x, info = dgfem.solve(out, out.rhs.reshape(-1), options=dgfem.solve_options(tolerance_scale=1e-4))
    exact = problems.function(capi.FN_SIN_SIN, (1.0,))
    err, h = dgfem.l2_error(x, dm, ref, exact)
    rp, col, val, rhs = orc.assemble(mesh.arrays(), ref.tables(), spec.c, p)
    xr, _ = onewton.direct_solve(*bsr_to_csr(rp, col, val), rhs.reshape(-1))
    sharp = dgfem.ReferenceElement(cfg.degree, capi.load().dgb_l2_quad_order(cfg.degree, cfg.quad_order))
    err_ref, h_ref = orc.l2_error(mesh.arrays(), sharp.tables(), xr, exact)
    assert abs(err - err_ref) <= 1e-8 * err_ref
    assert err < 1e-2   # P1 on 32^2: O(h^2) error of sin(pi x) sin(pi y)
