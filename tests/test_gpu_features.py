"""GPU: SpMV, error reporting, determinism, the host-buffer drop-in entry, shards, and
size-independent properties at full BASELINE sizes."""
import numpy as np
import pytest

from helpers import compare_system, gather_rows
from oracle.oracle import OracleLib, bsr_to_csr
from paper_1502_02941_b200 import capi, dgfem, problems, shard

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def oracle():
    return OracleLib()


def to_np(s):
    return (s.row_ptr.cpu().numpy(), s.col.cpu().numpy(), s.val.cpu().numpy(), s.rhs.cpu().numpy())


def test_inflow_on_neumann_reports_lowest_edge(oracle):
    """test_assembly.cpp:371-381, test_parallel_consistency.cpp:152-182."""
    mesh = dgfem.unit_square_mesh(6, 0.0, 0, False, 0, 15)   # all Neumann
    ref = dgfem.ReferenceElement(1)
    spec = problems.registry_get("smooth-sine")
    params = dgfem.set_parameters(capi.SIPG, 1)
    with pytest.raises(dgfem.Error) as e:
        dgfem.assemble_all(mesh, ref, spec, params)
    assert e.value.code == "InflowOnNeumann"
    from oracle.oracle import ReferenceError_
    with pytest.raises(ReferenceError_) as r:
        oracle.assemble(mesh.arrays(), ref.tables(), spec.c, params)
    assert e.value.detail == r.value.detail
    # the DROP policy assembles and matches the oracle's DROP
    params.neumann_inflow = capi.INFLOW_DROP
    g = dgfem.assemble_all(mesh, ref, spec, params)
    compare_system(to_np(g), oracle.assemble(mesh.arrays(), ref.tables(), spec.c, params))


def test_batch_reports_error_of_an_earlier_set(oracle):
    """dgb_assemble_batch over sets that differ in the Neumann policy (per-set launches): an
    InflowOnNeumann raised by the first set (ERROR) is still reported after a later set (DROP)
    assembled cleanly, with the reference's lowest-edge detail."""
    mesh = dgfem.unit_square_mesh(6, 0.0, 0, False, 0, 15)   # all Neumann
    ref = dgfem.ReferenceElement(1)
    spec = problems.registry_get("smooth-sine")
    p_err = dgfem.set_parameters(capi.SIPG, 1, capi.INFLOW_ERROR)
    p_drop = dgfem.set_parameters(capi.SIPG, 1, capi.INFLOW_DROP)
    a = shard.ShardAssembler(mesh, ref, spec, 0, 0, mesh.n_elements)
    b = shard.ShardAssembler(mesh, ref, spec, 0, 0, mesh.n_elements, share=a)
    with pytest.raises(dgfem.Error) as e:
        shard.assemble_batch([a, b], [p_err, p_drop])
    assert e.value.code == "InflowOnNeumann"
    from oracle.oracle import ReferenceError_
    with pytest.raises(ReferenceError_) as r:
        oracle.assemble(mesh.arrays(), ref.tables(), spec.c, p_err)
    assert e.value.detail == r.value.detail
    # a clean call afterwards reports no stale error
    shard.assemble_batch([a, b], [p_drop, p_drop])


def _l2_limit() -> int:
    from cuda.bindings import runtime as rt
    err, v = rt.cudaDeviceGetLimit(rt.cudaLimit.cudaLimitPersistingL2CacheSize)
    assert err == rt.cudaError_t.cudaSuccess
    return int(v)


def _set_l2_limit(v: int) -> None:
    from cuda.bindings import runtime as rt
    (err,) = rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitPersistingL2CacheSize, v)
    assert err == rt.cudaError_t.cudaSuccess


def test_l2_carve_out_is_restored():
    """The P1 plans' persisting-L2 carve-out is per device and reference counted: a bound plan
    raises the limit, the host-buffer entry (a cached plan) gives it back at the end of the
    call, and destroying the last plan restores the caller's own value."""
    import torch
    torch.cuda.init()
    cfg = problems.CONFIGS[4]
    mesh = dgfem.unit_square_mesh(64, 0.0, 0, True, 3, 0)
    ref = dgfem.ReferenceElement(cfg.degree, cfg.quad_order)
    spec = problems.config_problem(4)
    params = dgfem.config_parameters(cfg, capi.SIPG)
    _set_l2_limit(1 << 20)          # the caller's own carve-out
    start = _l2_limit()
    dgfem.assemble_all_host(mesh, ref.view, spec, params)
    assert _l2_limit() == start
    a = shard.ShardAssembler(mesh, ref, spec, 0, 0, mesh.n_elements, bind=True)
    b = shard.ShardAssembler(mesh, ref, spec, 0, 0, mesh.n_elements, bind=True)
    a.assemble(params)
    assert _l2_limit() >= start
    del a
    import gc
    gc.collect()
    assert _l2_limit() >= start    # b still holds its reference
    b.assemble(params)
    del b
    gc.collect()
    assert _l2_limit() == start
    _set_l2_limit(0)


@pytest.mark.parametrize("index", [2, 3])
def test_bitwise_reproducible(index):
    """No floating-point atomics: two runs give identical bits (test_parallel_consistency.cpp)."""
    import torch
    cfg = problems.CONFIGS[index]
    mesh = dgfem.unit_square_mesh(64, cfg.jitter, problems.SEED_JITTER, cfg.permute,
                                  problems.SEED_PERMUTE, cfg.neumann_sides)
    ref = dgfem.ReferenceElement(cfg.degree, cfg.quad_order)
    spec = problems.config_problem(index, mesh.n_elements)
    params = dgfem.config_parameters(cfg, cfg.methods[0])
    a = dgfem.assemble_all(mesh, ref, spec, params)
    b = dgfem.assemble_all(mesh, ref, spec, params)
    torch.cuda.synchronize()
    for x, y in zip((a.row_ptr, a.col, a.val, a.rhs), (b.row_ptr, b.col, b.val, b.rhs)):
        assert torch.equal(x, y)


def test_host_buffer_entry_matches_device_path(oracle):
    """dgb_assemble_all_host (the C-ABI call a reference maintainer binds) == device path."""
    import torch
    cfg = problems.CONFIGS[5]
    mesh = dgfem.unit_square_mesh(16, 0.0, 0, False, 0, 0)
    ref = dgfem.ReferenceElement(cfg.degree, cfg.quad_order)
    spec = problems.config_problem(5, mesh.n_elements)
    params = dgfem.config_parameters(cfg, capi.IIPG)
    h = dgfem.assemble_all_host(mesh, ref.view, spec, params)
    d = to_np(dgfem.assemble_all(mesh, ref, spec, params))
    torch.cuda.synchronize()
    for x, y in zip(h, d):
        np.testing.assert_array_equal(x, y)
    compare_system(h, oracle.assemble(mesh.arrays(), ref.tables(), spec.c, params))


def test_reference_tables_plan(oracle):
    """A plan built from the REFERENCE's own tables (golden dump), as in a drop-in deployment."""
    import os
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "tables.npz"))
    t = {k[len("k3_q7_"):]: z[k] for k in z.files if k.startswith("k3_q7_")}
    for k in ("degree", "n_local", "nq_vol", "nq_edge"):
        t[k] = int(t[k])
    cfg = problems.CONFIGS[3]
    mesh = dgfem.unit_square_mesh(10, cfg.jitter, problems.SEED_JITTER, False, 0, cfg.neumann_sides)
    spec = problems.config_problem(3)
    params = dgfem.config_parameters(cfg, capi.SIPG)
    view = dgfem.tables_struct(t)
    plan = dgfem.Plan(view)
    dm, dp = dgfem.DeviceMesh(mesh), dgfem.DeviceProblem(spec)
    out = plan.assemble(dm, dp, params, plan.allocate(dm))
    compare_system(to_np(out), oracle.assemble(mesh.arrays(), t, spec.c, params))


def test_shards_equal_full_assembly():
    """dgb_assemble_rows over a 3-way row split concatenates to dgb_assemble's output."""
    import torch
    cfg = problems.CONFIGS[2]
    mesh = dgfem.config_mesh(cfg, strips=3)
    ref = dgfem.ReferenceElement(cfg.degree, cfg.quad_order)
    spec = problems.config_problem(2, mesh.n_elements)
    params = dgfem.config_parameters(cfg, capi.NIPG)
    full = to_np(dgfem.assemble_all(mesh, ref, spec, params))
    parts, first = [], None
    for r in range(3):
        b, e = shard.row_range(mesh.n_elements, r, 3)
        sa = shard.ShardAssembler(mesh, ref, spec, 0, b, e, share=first)
        first = first or sa
        parts.append(to_np(sa.assemble(params)))
    torch.cuda.synchronize()
    off = np.cumsum([0] + [p[0][-1] for p in parts])
    rp = np.concatenate([p[0][:-1] + o for p, o in zip(parts, off)] + [[off[-1]]])
    np.testing.assert_array_equal(rp, full[0])
    for i in (1, 2, 3):
        np.testing.assert_array_equal(np.concatenate([p[i] for p in parts]), full[i])


def test_full_size_sipg_pure_diffusion_symmetric():
    """Config-3 mesh at full size (2.1 M triangles, P3) with b = 0, alpha = 0: K = D is
    symmetric to 1e-12 relative (acceptance.cpp criterion 5)."""
    import torch
    cfg = problems.CONFIGS[3]
    mesh = dgfem.config_mesh(cfg)
    ref = dgfem.ReferenceElement(cfg.degree, cfg.quad_order)
    spec = problems.config_problem(3)
    spec.c.advection = problems.vec_constant(0.0, 0.0)
    spec.c.linear_reaction = problems.constant(0.0)
    params = dgfem.config_parameters(cfg, capi.SIPG)
    s = dgfem.assemble_all(mesh, ref, spec, params)
    nl = ref.n_local
    E = mesh.n_elements
    rp = s.row_ptr.long()
    row_of_block = torch.repeat_interleave(torch.arange(E, device="cuda"), rp[1:] - rp[:-1])
    # transpose partner of block (e, f) is block (f, e): find it by a sort of (col, row) keys
    key = row_of_block * E + s.col.long()
    tkey = s.col.long() * E + row_of_block
    order = torch.argsort(key)
    pos = torch.searchsorted(key[order], tkey)
    partner = order[pos]
    assert torch.equal(key[partner], tkey)
    diff = (s.val - s.val[partner].transpose(1, 2)).abs().max().item()
    assert diff <= 1e-12 * s.val.abs().max().item()


def test_full_size_constant_annihilation_config2():
    """Config 2 at full size: for elements away from the boundary, K applied to the projection
    of u = 1 equals the reaction term alone (diffusion, penalty, consistency and upwind all
    annihilate constants; test_assembly.cpp:342-369)."""
    import torch
    cfg = problems.CONFIGS[2]
    mesh = dgfem.config_mesh(cfg)
    ref = dgfem.ReferenceElement(cfg.degree, cfg.quad_order)
    spec = problems.config_problem(2)
    params = dgfem.config_parameters(cfg, capi.SIPG)
    plan = dgfem.Plan(ref.view)
    dm, dp = dgfem.DeviceMesh(mesh), dgfem.DeviceProblem(spec)
    out = plan.assemble(dm, dp, params, plan.allocate(dm))
    nl = ref.n_local
    t = ref.tables()
    c0 = 1.0 / t["phi"].reshape(-1, nl)[0, 0]          # phi_0 is constant: u = 1 -> coef c0
    x = torch.zeros(mesh.n_elements * nl, dtype=torch.float64, device="cuda")
    x[0::nl] = c0
    y = torch.empty_like(x)
    plan.spmv(out, x, y)
    # reaction only: R x = det * alpha * M x, M = I: y_e = det_e * c0 on the first dof
    interior = torch.from_numpy(np.all(mesh.edge_kind[mesh.element_edges] == 0, axis=1)).cuda()
    nodes, el = mesh.nodes, mesh.elements
    p0, p1, p2 = nodes[el[:, 0]], nodes[el[:, 1]], nodes[el[:, 2]]
    det = (p1[:, 0] - p0[:, 0]) * (p2[:, 1] - p0[:, 1]) - (p2[:, 0] - p0[:, 0]) * (p1[:, 1] - p0[:, 1])
    expect = torch.zeros_like(y).view(-1, nl)
    expect[:, 0] = torch.from_numpy(det).cuda() * c0
    err = (y.view(-1, nl) - expect)[interior].abs().max().item()
    assert err <= 1e-12 * (c0 * 18.0 * 1e-4 * 4)  # << penalty / diffusion scale of the entries


def test_config1_solve_error(oracle):
    """Config 1's own check: solve K u = F on the CPU (scipy; the reference's Eigen solver is
    absent) and compare the L2 error with the exact solution against the oracle system's."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla
    cfg = problems.CONFIGS[1]
    mesh = dgfem.config_mesh(cfg)
    ref = dgfem.ReferenceElement(cfg.degree, cfg.quad_order)
    spec = problems.config_problem(1)
    params = dgfem.config_parameters(cfg, capi.SIPG)
    t = ref.tables()

    def l2_error(rp, col, val, rhs):
        crp, ccol, cval = bsr_to_csr(rp, col, val)
        n = crp.shape[0] - 1
        u = spla.spsolve(sp.csr_matrix((cval, ccol, crp), shape=(n, n)).tocsc(), rhs.reshape(-1))
        nl = t["n_local"]
        phi = t["phi"].reshape(-1, nl)
        nodes, el = mesh.nodes, mesh.elements
        p0, p1, p2 = nodes[el[:, 0]], nodes[el[:, 1]], nodes[el[:, 2]]
        B = np.stack([p1 - p0, p2 - p0], axis=2)                 # [E, 2, 2]
        det = np.abs(np.linalg.det(B))
        xq = p0[:, None, :] + np.einsum("eij,qj->eqi", B, np.stack([t["vol_x"], t["vol_y"]], 1))
        uh = u.reshape(-1, nl) @ phi.T                            # [E, q]
        ue = np.sin(np.pi * xq[..., 0]) * np.sin(np.pi * xq[..., 1])
        return np.sqrt(np.sum(det[:, None] * t["vol_w"][None, :] * (uh - ue) ** 2))

    e_gpu = l2_error(*to_np(dgfem.assemble_all(mesh, ref, spec, params)))
    e_orc = l2_error(*oracle.assemble(mesh.arrays(), t, spec.c, params))
    assert e_gpu < 5e-3
    assert abs(e_gpu - e_orc) <= 1e-9 * e_orc


def test_bound_pattern_single_kernel_matches_unbound():
    """dgb_plan_bind_mesh: the one-kernel path equals the count+scan path bitwise, for the full
    mesh and for a shard; unbinding falls back."""
    import torch
    cfg = problems.CONFIGS[2]
    mesh = dgfem.unit_square_mesh(40, 0.1, 3, True, 4, 0)
    ref = dgfem.ReferenceElement(cfg.degree, cfg.quad_order)
    spec = problems.config_problem(2)
    params = dgfem.config_parameters(cfg, capi.IIPG)
    plan = dgfem.Plan(ref.view)
    plan.set_option(capi.OPTION_WARP_SPECIALIZED, 0)  # same kernel body bound / unbound
    dm, dp = dgfem.DeviceMesh(mesh), dgfem.DeviceProblem(spec)
    a = plan.assemble(dm, dp, params, plan.allocate(dm))
    assert capi.load().dgb_plan_launch_count(plan._h) == 4
    plan.bind_mesh(dm)
    b = plan.allocate(dm)
    b.row_ptr.fill_(-7)
    plan.assemble(dm, dp, params, b)
    assert capi.load().dgb_plan_launch_count(plan._h) == 1
    torch.cuda.synchronize()
    for x, y in zip((a.row_ptr, a.col, a.val, a.rhs), (b.row_ptr, b.col, b.val, b.rhs)):
        assert torch.equal(x, y)
    # shard with its own bound pattern
    lo, hi = shard.row_range(mesh.n_elements, 1, 3)
    sa = shard.ShardAssembler(mesh, ref, spec, 0, lo, hi, bind=True)
    sa.plan.set_option(capi.OPTION_WARP_SPECIALIZED, 0)
    out = sa.assemble(params)
    full = to_np(a)
    part = to_np(out)
    np.testing.assert_array_equal(part[0], full[0][lo:hi + 1] - full[0][lo])
    np.testing.assert_array_equal(part[2], full[2][full[0][lo]:full[0][hi]])
    capi.load().dgb_plan_unbind_mesh(plan._h)
    plan.assemble(dm, dp, params, b)
    assert capi.load().dgb_plan_launch_count(plan._h) == 4


@pytest.mark.parametrize("fuse", [True, False])
@pytest.mark.parametrize("cfg_index", [2, 3, 4])
def test_batch_equals_separate_assemblies(cfg_index, fuse):
    """dgb_assemble_batch (SIPG, NIPG, IIPG in one launch for the tensor-core kernels on a
    bound mesh; a loop otherwise) writes what three dgb_assemble_rows calls write.  Fused
    (each CTA writes every set from one per-element pass): pattern bitwise, K and F within
    rounding (kappa is applied to a separate product / RHS part)."""
    cfg = problems.CONFIGS[cfg_index]
    mesh = dgfem.unit_square_mesh(48, cfg.jitter, problems.SEED_JITTER, cfg.permute,
                                  problems.SEED_PERMUTE, cfg.neumann_sides)
    ref = dgfem.ReferenceElement(cfg.degree, cfg.quad_order)
    spec = problems.config_problem(cfg_index, mesh.n_elements)
    methods = [capi.SIPG, capi.NIPG, capi.IIPG]
    params = [dgfem.config_parameters(cfg, m) for m in methods]
    a = [shard.ShardAssembler(mesh, ref, spec, 0, 0, mesh.n_elements, bind=True)]
    a += [shard.ShardAssembler(mesh, ref, spec, 0, 0, mesh.n_elements, share=a[0]) for _ in methods[1:]]
    a[0].plan.set_option(capi.OPTION_BATCH_FUSE, int(fuse))
    shard.assemble_batch(a, params)
    got = [to_np(x.out) for x in a]
    for p, g in zip(params, got):
        single = shard.ShardAssembler(mesh, ref, spec, 0, 0, mesh.n_elements, share=a[0])
        want = to_np(single.assemble(p))
        for x, y in zip(g[:2], want[:2]):
            assert np.array_equal(x, y)
        # K, F: rounding-level differences (fused: kappa applied to a separate product / RHS
        # part; single P-form assemblies run the warp-specialised kernel, whose per-element
        # pass the compiler contracts into FMAs differently)
        for x, y in zip(g[2:], want[2:]):
            np.testing.assert_allclose(x, y, rtol=0, atol=1e-14 * np.abs(y).max())


def test_batch_mixed_penalties_not_fused():
    """Sets whose penalties differ cannot share the per-element pass: the batch still matches
    the separate assemblies bitwise (one CTA row per set)."""
    cfg = problems.CONFIGS[2]
    mesh = dgfem.unit_square_mesh(40)
    ref = dgfem.ReferenceElement(cfg.degree, cfg.quad_order)
    spec = problems.config_problem(2, mesh.n_elements)
    params = [dgfem.config_parameters(cfg, m) for m in (capi.SIPG, capi.NIPG)]
    params[1].sigma_interior *= 2.0
    a = [shard.ShardAssembler(mesh, ref, spec, 0, 0, mesh.n_elements, bind=True)]
    a.append(shard.ShardAssembler(mesh, ref, spec, 0, 0, mesh.n_elements, share=a[0]))
    shard.assemble_batch(a, params)
    for p, x in zip(params, a):
        single = shard.ShardAssembler(mesh, ref, spec, 0, 0, mesh.n_elements, share=a[0])
        for u, v in zip(to_np(x.out), to_np(single.assemble(p))):
            assert np.array_equal(u, v)


@pytest.mark.parametrize("degree", [2, 3])
@pytest.mark.parametrize("batch", [False, True])
def test_warp_specialized_equals_monolithic(degree, batch):
    """The persistent producer / consumer kernel (assemble_ws.cuh; P-form tensor-core configs
    on a bound mesh) writes what the monolithic kernel writes -- the pattern bitwise, K and F
    to rounding (FMA contraction differs) -- for single assemblies and fused batches;
    77 x 77 cells: a ragged last chunk and uneven chunks per pair, Neumann sides included."""
    cfg = problems.CONFIGS[2]
    mesh = dgfem.unit_square_mesh(77, 0.2, problems.SEED_JITTER, True, problems.SEED_PERMUTE,
                                  problems.CONFIGS[3].neumann_sides)
    ref = dgfem.ReferenceElement(degree, 2 * degree)
    spec = problems.config_problem(2, mesh.n_elements)
    methods = [capi.SIPG, capi.NIPG, capi.IIPG] if batch else [capi.NIPG]
    params = [dgfem.config_parameters(cfg, m) for m in methods]
    got = {}
    for ws in (8, 0):  # 8: forced on (8 producer warps), also for single assemblies
        a = [shard.ShardAssembler(mesh, ref, spec, 0, 0, mesh.n_elements, bind=True)]
        a += [shard.ShardAssembler(mesh, ref, spec, 0, 0, mesh.n_elements, share=a[0]) for _ in methods[1:]]
        a[0].plan.set_option(capi.OPTION_WARP_SPECIALIZED, ws)
        if batch:
            shard.assemble_batch(a, params)
        else:
            a[0].assemble(params[0])
        got[ws] = [to_np(x.out) for x in a]
    for x, y in zip(got[8], got[0]):
        for u, v in zip(x[:2], y[:2]):
            assert np.array_equal(u, v)
        for u, v in zip(x[2:], y[2:]):
            np.testing.assert_allclose(u, v, rtol=0, atol=1e-14 * np.abs(v).max())


@pytest.mark.parametrize("rows", [None, (1, 3)])
def test_p1_persistent_kernel_equals_one_shot(oracle, rows):
    """The persistent software-pipelined P1 kernel (DGB_OPTION_P1_PIPELINE, default), with the
    auto L2 policy (evict-last node gathers in a persisting carve-out) and
    with plain evict-first output, writes what the one-shot P1 kernel writes and what the
    unbound path writes: the pattern bitwise, K and F to rounding.  Permuted, jittered mesh
    (a ragged last chunk), full mesh and a shard."""
    import torch
    cfg = problems.CONFIGS[4]
    mesh = dgfem.unit_square_mesh(45, 0.2, problems.SEED_JITTER, True, problems.SEED_PERMUTE)
    ref = dgfem.ReferenceElement(cfg.degree, cfg.quad_order)
    spec = problems.config_problem(4, mesh.n_elements)
    params = dgfem.config_parameters(cfg, capi.SIPG)
    lo, hi = (0, mesh.n_elements) if rows is None else shard.row_range(mesh.n_elements, *rows)
    got = {}
    for key, pipe, l2 in (("pipe12", 1, -1), ("pipe12_ef", 1, 2),
                          ("oneshot", 0, -1), ("unbound", 1, -1)):
        a = shard.ShardAssembler(mesh, ref, spec, 0, lo, hi, bind=False)
        a.plan.set_option(capi.OPTION_L2_POLICY, l2)
        a.plan.set_option(capi.OPTION_P1_PIPELINE, pipe)
        if key != "unbound":
            a.plan.bind_mesh(a.dmesh, lo, hi)
        got[key] = to_np(a.assemble(params))
        torch.cuda.synchronize()
    base = got["oneshot"]
    for key, x in got.items():
        np.testing.assert_array_equal(x[0], base[0])
        np.testing.assert_array_equal(x[1], base[1])
        for u, v in zip(x[2:], base[2:]):
            np.testing.assert_allclose(u, v, rtol=0, atol=1e-13 * np.abs(v).max())
    # and the whole thing against the oracle (full mesh)
    if rows is None:
        rp, col, val, rhs = oracle.assemble(mesh.arrays(), ref.tables(), spec.c, params)
        assert np.array_equal(base[0], rp) and np.array_equal(base[1], col)
        assert np.abs(got["pipe12"][2] - val).max() <= 1e-12 * np.abs(val).max()


P1_SOURCES = {
    "constant": lambda: problems.constant(1.5),
    "sine": lambda: problems.source_of(capi.FN_SIN_SIN, (1.0,), alpha=1.0, eps=0.05, bx=0.8, by=-0.3),
    "gaussian": lambda: problems.source_of(capi.FN_GAUSSIAN, (50.0, 0.5, 0.5), alpha=1.0, eps=0.05,
                                           bx=0.8, by=-0.3),
    "tanh": lambda: problems.source_of(capi.FN_TANH_LAYER, (1.0, -1.0, -0.25, 0.1), alpha=1.0, eps=0.05,
                                       bx=0.8, by=-0.3),
}
P1_DIRICHLET = {
    "constant": lambda: problems.constant(0.25),
    "sine": lambda: problems.function(capi.FN_SIN_SIN, (1.0,)),
    "gaussian": lambda: problems.function(capi.FN_GAUSSIAN, (50.0, 0.5, 0.5)),
    "tanh": lambda: problems.function(capi.FN_TANH_LAYER, (1.0, -1.0, -0.25, 0.1)),
}


@pytest.mark.parametrize("family", sorted(P1_SOURCES))
def test_p1_bound_kernel_every_source_family(oracle, family):
    """The persistent P1 kernel is compiled once per source family (constant / per-element, sine
    product, Gaussian, any other) and reads its geometry from the record bound per chunk; boundary
    data go through the branch-free cores.  Every instantiation, with the geometry record, with
    the node gathers (DGB_OPTION_GEOMETRY_CACHE 0) and unbound, against the oracle with the
    per-row comparator -- jittered permuted mesh, Neumann sides, per-element eps and alpha."""
    import torch
    cfg = problems.CONFIGS[1]
    mesh = dgfem.unit_square_mesh(37, 0.2, 21, True, 22, 2)
    ref = dgfem.ReferenceElement(cfg.degree, cfg.quad_order)
    spec = problems.make_problem("p1-" + family, 0.05, problems.vec_constant(0.8, -0.3), 1.0,
                                 P1_SOURCES[family](), P1_DIRICHLET[family](), neumann_sides=2)
    r = problems.uniform01(4242, 2 * mesh.n_elements)
    spec.set_per_element("diffusion", 10.0 ** (-3.0 + 3.0 * r[:mesh.n_elements]))
    spec.set_per_element("linear_reaction", 2.0 * r[mesh.n_elements:])
    params = dgfem.set_parameters(capi.SIPG, cfg.degree, capi.INFLOW_DROP)
    want = oracle.assemble(mesh.arrays(), ref.tables(), spec.c, params)
    got = {}
    for key, geo, bind in (("record", 1, True), ("gathers", 0, True), ("unbound", 1, False)):
        a = shard.ShardAssembler(mesh, ref, spec, 0, 0, mesh.n_elements, bind=False)
        a.plan.set_option(capi.OPTION_GEOMETRY_CACHE, geo)
        if bind:
            a.plan.bind_mesh(a.dmesh, 0, mesh.n_elements)
        got[key] = to_np(a.assemble(params))
        torch.cuda.synchronize()
        compare_system(got[key], want)
    # the record holds the values the gathering kernel computes itself; the instantiations
    # differ only in the compiler's FMA contraction (last bits)
    for u, v in zip(got["record"][2:], got["gathers"][2:]):
        np.testing.assert_allclose(u, v, rtol=0, atol=1e-13 * np.abs(v).max())
