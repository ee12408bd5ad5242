"""GPU parity: the sm_100a assembly vs the C restatement oracle (pinned bitwise to the
reference), through the C-ABI.  Comparator: SURVEY.md §8(c)."""
import numpy as np
import pytest

from helpers import compare_system, gather_rows
from oracle.oracle import OracleLib
from paper_1502_02941_b200 import capi, dgfem, problems

pytestmark = pytest.mark.gpu

REGISTRY = ["smooth-sine", "smooth-sine-mixed", "poly-exact", "paper-boundary-layer-linear",
            "paper-boundary-layer",
            "pure-advection-patch"]


@pytest.fixture(scope="module")
def oracle():
    return OracleLib()


def run_gpu(mesh, ref, spec, params):
    import torch
    s = dgfem.assemble_all(mesh, ref, spec, params)
    torch.cuda.synchronize()
    return (s.row_ptr.cpu().numpy(), s.col.cpu().numpy(), s.val.cpu().numpy(),
            s.rhs.cpu().numpy())


@pytest.mark.parametrize("name", REGISTRY)
@pytest.mark.parametrize("degree", [1, 2, 3, 4])
def test_registry_problems(oracle, name, degree):
    spec = problems.registry_get(name)
    mesh = dgfem.unit_square_mesh(6, 0.15, 11, True, 12, spec.neumann_sides)
    ref = dgfem.ReferenceElement(degree)
    for method in (capi.SIPG, capi.NIPG, capi.IIPG):
        params = dgfem.set_parameters(method, degree)
        g = run_gpu(mesh, ref, spec, params)
        o = oracle.assemble(mesh.arrays(), ref.tables(), spec.c, params)
        compare_system(g, o)


@pytest.mark.parametrize("index", [1, 2, 3, 4, 5])
def test_configs_small(oracle, index):
    cfg = problems.CONFIGS[index]
    n = 12
    mesh = dgfem.unit_square_mesh(n, cfg.jitter, problems.SEED_JITTER, cfg.permute,
                                  problems.SEED_PERMUTE, cfg.neumann_sides)
    ref = dgfem.ReferenceElement(cfg.degree, cfg.quad_order)
    spec = problems.config_problem(index, mesh.n_elements)
    for method in cfg.methods:
        params = dgfem.config_parameters(cfg, method)
        g = run_gpu(mesh, ref, spec, params)
        o = oracle.assemble(mesh.arrays(), ref.tables(), spec.c, params)
        compare_system(g, o)


@pytest.mark.parametrize("index", [1, 2, 3, 4, 5])
def test_configs_full_size_sampled_rows(oracle, index):
    """Full BASELINE.json sizes; the oracle recomputes a seeded sample of block rows."""
    cfg = problems.CONFIGS[index]
    mesh = dgfem.config_mesh(cfg)
    ref = dgfem.ReferenceElement(cfg.degree, cfg.quad_order)
    spec = problems.config_problem(index, mesh.n_elements)
    rng = np.random.default_rng(1000 + index)
    rows = np.unique(np.concatenate([
        rng.choice(mesh.n_elements, size=min(mesh.n_elements, 4000), replace=False),
        np.arange(min(64, mesh.n_elements)), np.arange(mesh.n_elements - 64, mesh.n_elements)]))
    for method in cfg.methods:
        params = dgfem.config_parameters(cfg, method)
        g = run_gpu(mesh, ref, spec, params)
        assert g[0][-1] == mesh.n_elements + 2 * mesh.n_interior_edges
        o = oracle.assemble(mesh.arrays(), ref.tables(), spec.c, params, rows=rows)
        compare_system(gather_rows(*g, rows), o)


@pytest.mark.parametrize("index", [1, 2, 3, 4, 5])
def test_generic_kernel_matches_oracle(oracle, index):
    """The generic (any quadrature) block-row kernel stays parity-green too."""
    import torch
    cfg = problems.CONFIGS[index]
    mesh = dgfem.unit_square_mesh(10, cfg.jitter, problems.SEED_JITTER, cfg.permute,
                                  problems.SEED_PERMUTE, cfg.neumann_sides)
    ref = dgfem.ReferenceElement(cfg.degree, cfg.quad_order)
    spec = problems.config_problem(index, mesh.n_elements)
    params = dgfem.config_parameters(cfg, cfg.methods[-1])
    s = dgfem.assemble_all(mesh, ref, spec, params, generic=True)
    torch.cuda.synchronize()
    g = (s.row_ptr.cpu().numpy(), s.col.cpu().numpy(), s.val.cpu().numpy(), s.rhs.cpu().numpy())
    compare_system(g, oracle.assemble(mesh.arrays(), ref.tables(), spec.c, params))


def test_velocity_kinds_on_p1(oracle):
    """Constant, affine and trigonometric velocities through the specialised P1 kernels."""
    mesh = dgfem.unit_square_mesh(9, 0.2, 5, True, 6, 0)
    ref = dgfem.ReferenceElement(1, 3)
    for b in (problems.vec_constant(0.3, -0.7), problems.vec_affine(0.5, -0.5, 0.0, -1.0, 1.0, 0.0),
              problems.vec_trig(2 * problems.PI, 2 * problems.PI)):
        spec = problems.config_problem(1)
        spec.c.advection = b
        for method in (capi.SIPG, capi.NIPG, capi.IIPG):
            params = dgfem.set_parameters(method, 1)
            compare_system(run_gpu(mesh, ref, spec, params),
                           oracle.assemble(mesh.arrays(), ref.tables(), spec.c, params))


# Every specialised kernel -- (degree, quad_order) -> (nl, nq_vol, nq_edge) -- with each velocity
# kind it is built for, per-element eps / alpha (the edge average of eps, element alpha), a
# Neumann side (outflow-only convention), every method, on a jittered permuted mesh.
KERNEL_CASES = [
    (1, 3, "const"), (1, 3, "affine"), (1, 3, "trig"),   # P1 stash-free / general kernels
    (2, 5, "const"), (2, 6, "const"),                    # P2 tensor cores (P-form)
    (3, 7, "const"), (3, 7, "affine"),                   # P3 tensor cores (P-form, U-form)
    (4, 9, "trig"),                                      # P4 tensor cores (T-form)
    (2, 5, "affine"), (3, 7, "trig"),                    # generic kernel
]


@pytest.mark.parametrize("degree,quad_order,vel", KERNEL_CASES)
def test_every_kernel_per_element_fields(oracle, degree, quad_order, vel):
    mesh = dgfem.unit_square_mesh(10, 0.2, 31, True, 32, 2)
    ref = dgfem.ReferenceElement(degree, quad_order)
    b = {"const": problems.vec_constant(0.8, -0.3),
         "affine": problems.vec_affine(0.5, -0.5, 0.0, -1.0, 1.0, 0.0),
         "trig": problems.vec_trig(2 * problems.PI, 2 * problems.PI)}[vel]
    u = (capi.FN_SIN_SIN, (1.0,))
    spec = problems.make_problem("kernels", 1.0, b, 1.0, problems.function(*u),
                                 problems.function(*u), neumann_sides=2)
    r = problems.uniform01(777 + degree, 2 * mesh.n_elements)
    spec.set_per_element("diffusion", 10.0 ** (-4.0 + 4.0 * r[:mesh.n_elements]))
    spec.set_per_element("linear_reaction", 2.0 * r[mesh.n_elements:])
    for method in (capi.SIPG, capi.NIPG, capi.IIPG):
        params = dgfem.set_parameters(method, degree, capi.INFLOW_DROP)
        g = run_gpu(mesh, ref, spec, params)
        o = oracle.assemble(mesh.arrays(), ref.tables(), spec.c, params)
        compare_system(g, o)


@pytest.mark.parametrize("level,degree", [(3, 1), (3, 2), (4, 1)])
def test_reference_benchmark_cases(oracle, level, degree):
    """The reference's own assembly benchmark (bench/assembly_bench.cpp:31-48, configure :79-93):
    unit_square_mesh refined `level` times, build_reference(k), paper-boundary-layer (with its
    f += u^2 source), SIPG -- the mesh built and refined on the device, the assembly through the
    GPU path, compared with the oracle on the same arrays."""
    import torch
    from test_solve_oracle import UNIT_SQUARE
    raw = UNIT_SQUARE
    m = dgfem.device_build_mesh(raw["nodes"], raw["elements"], raw["dirichlet"], raw["neumann"])
    for _ in range(level):
        m = m.refine()
    spec = problems.registry_get("paper-boundary-layer")
    ref = dgfem.ReferenceElement(degree)
    params = dgfem.set_parameters(capi.SIPG, degree)
    plan = dgfem.Plan(ref.view)
    out = plan.assemble(m, dgfem.DeviceProblem(spec), params, plan.allocate(m))
    torch.cuda.synchronize()
    g = (out.row_ptr.cpu().numpy(), out.col.cpu().numpy(), out.val.cpu().numpy(), out.rhs.cpu().numpy())
    compare_system(g, oracle.assemble(m.arrays(), ref.tables(), spec.c, params))
