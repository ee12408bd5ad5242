"""GPU BSR SpMV (csrc/spmv.cu) against the oracle's matvec restatement (the reference's
`matvec`, sparse.cpp:116-129, on stiffness()'s CSR): |dy_i| <= 1e-12 sum_j |K_ij x_j|
(SURVEY.md §8(c))."""
import numpy as np
import pytest

from oracle.oracle import OracleLib
from paper_1502_02941_b200 import capi, dgfem, problems, workload

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def oracle():
    return OracleLib()


def _check(oracle, rp, col, val, x, y):
    y_ref = oracle.spmv(rp, col, val, x)
    scale = oracle.spmv(rp, col, np.abs(val), np.abs(x))
    err = np.abs(y - y_ref)
    assert np.all(err <= 1e-12 * scale + 1e-300), float((err / np.maximum(scale, 1e-300)).max())


def test_config4_hundred_products(oracle):
    """Config 4 at full size (8.4M block rows, 33.5M blocks): the bench's 100 products on the
    seeded U[-1,1] x; the first checked against the oracle, all 100 bitwise identical."""
    import torch
    sp = workload.SpmvRun(4)
    stream = torch.cuda.current_stream(0)
    sp.step(stream)
    torch.cuda.synchronize()
    first = sp.y.clone()
    for _ in range(99):
        sp.step(stream)
    torch.cuda.synchronize()
    assert torch.equal(first, sp.y)
    s = sp.system
    _check(oracle, s.row_ptr.cpu().numpy(), s.col.cpu().numpy(), s.val.cpu().numpy(),
           sp.x.cpu().numpy(), first.cpu().numpy())


@pytest.mark.parametrize("index", [1, 2, 3, 5])
def test_every_block_size(oracle, index):
    """nl = 3, 6, 10, 15 on the config's coefficients (small permuted meshes: ragged tiles)."""
    import torch
    cfg = problems.CONFIGS[index]
    mesh = dgfem.unit_square_mesh(23, cfg.jitter, 5, True, 6, cfg.neumann_sides)
    ref = dgfem.ReferenceElement(cfg.degree, cfg.quad_order)
    spec = problems.config_problem(index, mesh.n_elements)
    s = dgfem.assemble_all(mesh, ref, spec, dgfem.config_parameters(cfg, cfg.methods[0]))
    n = mesh.n_elements * ref.n_local
    x = torch.from_numpy(2.0 * problems.uniform01(index, n) - 1.0).cuda()
    y = torch.full_like(x, float("nan"))
    dgfem.Plan(ref.view).spmv(s, x, y)
    torch.cuda.synchronize()
    _check(oracle, s.row_ptr.cpu().numpy(), s.col.cpu().numpy(), s.val.cpu().numpy(),
           x.cpu().numpy(), y.cpu().numpy())


def _random_bsr(n_rows, nl, max_per_row, seed):
    rng = np.random.default_rng(seed)
    counts = rng.integers(0, max_per_row + 1, n_rows)
    rp = np.zeros(n_rows + 1, np.int32)
    rp[1:] = np.cumsum(counts)
    col = np.concatenate([np.sort(rng.choice(n_rows, c, replace=False)) for c in counts]).astype(np.int32)
    val = rng.uniform(-1, 1, (rp[-1], nl, nl))
    return rp, col, val


@pytest.mark.parametrize("nl", [3, 6, 10, 15])
@pytest.mark.parametrize("max_per_row,unaligned", [(4, False), (12, False), (4, True)])
def test_general_bsr(oracle, nl, max_per_row, unaligned):
    """Any valid BSR: rows with more blocks than the staged capacity (global path), empty
    rows, and a value array that is not 16-byte aligned."""
    import torch
    rp, col, val = _random_bsr(1000, nl, max_per_row, 7 * nl + max_per_row)
    dev = torch.device("cuda", 0)
    flat = torch.zeros(val.size + 1, dtype=torch.float64, device=dev)
    tv = flat[1:] if unaligned else flat[:-1]
    tv.copy_(torch.from_numpy(val.reshape(-1)))
    b = capi.Bsr()
    b.n_block_rows, b.block_dim, b.nnzb = 1000, nl, col.size
    trp, tcol = torch.from_numpy(rp).to(dev), torch.from_numpy(col).to(dev)
    b.row_ptr, b.col, b.val = trp.data_ptr(), tcol.data_ptr(), tv.data_ptr()
    x = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, 1000 * nl)).to(dev)
    y = torch.full_like(x, float("nan"))
    import ctypes as C
    dgfem._check(capi.load().dgb_spmv(C.byref(b), x.data_ptr(), y.data_ptr(), None))
    torch.cuda.synchronize()
    _check(oracle, rp, col, val, x.cpu().numpy(), y.cpu().numpy())


def test_empty_matrix():
    import ctypes as C
    b = capi.Bsr()
    b.n_block_rows, b.block_dim, b.nnzb = 0, 3, 0
    dgfem._check(capi.load().dgb_spmv(C.byref(b), 8, 8, None))  # nothing is touched
