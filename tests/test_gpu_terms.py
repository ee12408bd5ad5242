"""GPU per-term assembly (dgb_assemble_terms) against the reference's own D, C and R
(assemble_diffusion / assemble_convection / assemble_reaction, assembly.hpp:72-95), and the
reference's per-term property tests on the GPU path: bitwise-level SIPG symmetry of D
(test_assembly.cpp:263-279, acceptance.cpp criterion 5) and mass blocks = det I
(test_assembly.cpp:383-406, acceptance.cpp criterion 6)."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle.oracle import RefLib, bsr_to_csr
from paper_1502_02941_b200 import capi, dgfem, problems

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    try:
        return RefLib()
    except FileNotFoundError:
        pytest.skip("oracle/_ref (the compiled reference) is not built")


def gpu_terms(mesh, refel, spec, params, terms):
    import torch
    plan = dgfem.Plan(refel.view)
    dm, dp = dgfem.DeviceMesh(mesh), dgfem.DeviceProblem(spec)
    out = plan.assemble_terms(dm, dp, params, terms, plan.allocate(dm))
    torch.cuda.synchronize()
    rp, col, val = out.row_ptr.cpu().numpy(), out.col.cpu().numpy(), out.val.cpu().numpy()
    ro, ci, va = bsr_to_csr(rp, col, val)
    n = (rp.shape[0] - 1) * val.shape[1]
    return sp.csr_matrix((va, ci, ro), shape=(n, n))


def assert_close(g, r, tol=1e-12):
    d = (g - r).tocsr()
    scale = np.maximum(abs(r).max(axis=1).toarray().ravel(), abs(g).max(axis=1).toarray().ravel())
    err = abs(d).max(axis=1).toarray().ravel()
    worst = float((err / np.maximum(scale, 1e-300)).max()) if err.size else 0.0
    assert worst <= tol, worst


@pytest.mark.parametrize("index", [1, 2, 3, 4, 5])
def test_terms_match_reference_D_C_R(ref, index):
    """Config coefficients on a 10x10 mesh: each GPU term equals the reference's matrix of that
    term (entries of K's pattern outside the term's own pattern are exact zeros); D + C + R
    equals the full assembly."""
    cfg = problems.CONFIGS[index]
    mesh = dgfem.unit_square_mesh(10, cfg.jitter, problems.SEED_JITTER, cfg.permute,
                                  problems.SEED_PERMUTE, cfg.neumann_sides)
    refel = dgfem.ReferenceElement(cfg.degree, cfg.quad_order)
    spec = problems.config_problem(index, mesh.n_elements)
    params = dgfem.config_parameters(cfg, cfg.methods[-1])
    raw = mesh.raw()
    rmesh = ref.build_mesh(raw["nodes"], raw["elements"], raw["dirichlet"], raw["neumann"])
    rp = ref.set_parameters(params.method, cfg.degree)
    rp.sigma_interior, rp.sigma_boundary = params.sigma_interior, params.sigma_boundary
    clip = cfg.neumann_sides if cfg.neumann_inflow == capi.INFLOW_DROP else 0
    system = ref.assemble(rmesh, ref.reference(cfg.degree, cfg.quad_order), spec.c, rp, clip_sides=clip)
    n = mesh.n_elements * refel.n_local
    mats = {}
    for which, term in ((1, capi.TERM_DIFFUSION), (2, capi.TERM_CONVECTION), (3, capi.TERM_REACTION)):
        ro, ci, va = system.csr(which)
        r = sp.csr_matrix((va, ci, ro), shape=(n, n))
        g = gpu_terms(mesh, refel, spec, params, term)
        assert_close(g, r)
        mats[term] = g
    full = gpu_terms(mesh, refel, spec, params, capi.TERM_ALL)
    assert_close((mats[1] + mats[2]) + mats[4], full)


@pytest.mark.parametrize("degree", [1, 2, 3, 4])
def test_sipg_diffusion_symmetric(degree):
    """SIPG D is symmetric (test_assembly.cpp:263-279): ||D - D^T||_F <= 1e-12 ||D||_F."""
    spec = problems.registry_get("smooth-sine")
    mesh = dgfem.unit_square_mesh(8, 0.2, 3, True, 4)
    refel = dgfem.ReferenceElement(degree)
    D = gpu_terms(mesh, refel, spec, dgfem.set_parameters(capi.SIPG, degree), capi.TERM_DIFFUSION)
    assert sp.linalg.norm(D - D.T) <= 1e-12 * sp.linalg.norm(D)


@pytest.mark.parametrize("degree", [1, 2, 3, 4])
def test_mass_blocks_are_det_identity(degree):
    """alpha = 1: every reaction block is det(B) I for the orthonormal Dubiner basis
    (test_assembly.cpp:383-406, acceptance.cpp criterion 6)."""
    spec = problems.registry_get("smooth-sine")
    mesh = dgfem.unit_square_mesh(6, 0.2, 5, True, 6)
    refel = dgfem.ReferenceElement(degree)
    R = gpu_terms(mesh, refel, spec, dgfem.set_parameters(capi.SIPG, degree), capi.TERM_REACTION)
    nl = refel.n_local
    a = mesh.arrays()
    p = a["nodes"][a["elements"]]
    det = (p[:, 1, 0] - p[:, 0, 0]) * (p[:, 2, 1] - p[:, 0, 1]) - (p[:, 2, 0] - p[:, 0, 0]) * (p[:, 1, 1] - p[:, 0, 1])
    Rd = R.toarray()
    for e in range(mesh.n_elements):
        blk = Rd[e * nl:(e + 1) * nl, e * nl:(e + 1) * nl]
        assert np.abs(blk - det[e] * np.eye(nl)).max() <= 1e-12 * abs(det[e])
    # and nothing off the block diagonal
    off = R.copy().tolil()
    for e in range(mesh.n_elements):
        off[e * nl:(e + 1) * nl, e * nl:(e + 1) * nl] = 0
    assert abs(off.tocsr()).max() == 0.0


def test_terms_mask_validation():
    mesh = dgfem.unit_square_mesh(2)
    refel = dgfem.ReferenceElement(1)
    plan = dgfem.Plan(refel.view)
    dm, dp = dgfem.DeviceMesh(mesh), dgfem.DeviceProblem(problems.registry_get("smooth-sine"))
    with pytest.raises(dgfem.Error):
        plan.assemble_terms(dm, dp, dgfem.set_parameters(capi.SIPG, 1), 9, plan.allocate(dm))
