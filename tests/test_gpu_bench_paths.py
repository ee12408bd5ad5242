"""Full-size parity of the exact launches `bench.py` times ("Next round" 1).

Every number in a bench line comes from `workload.ConfigRun.step()`: a bound mesh
(`dgb_plan_bind_mesh`), the library's default kernel choice and L2 policy, and for config 2 the
fused warp-specialised `dgb_assemble_batch` of all three methods.  These tests run that same
object at the BASELINE.json sizes and compare with the oracle (pinned bitwise to the reference,
tests/test_oracle_golden.py) under SURVEY.md §8(c)'s comparator:

* the whole BSR pattern bit-exact against the pattern derived from the mesh (every row);
* >= 4,000 seeded block rows plus the first and last 64 recomputed by the oracle: every K entry
  within 1e-12 of its row's max, every F entry within 1e-12 of its element block's max.
"""
import numpy as np
import pytest

from helpers import compare_system, expected_pattern, gather_rows_device, sample_rows
from oracle.oracle import OracleLib
from paper_1502_02941_b200 import workload

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def oracle():
    return OracleLib()


def _check_run(oracle, run, seed):
    import torch
    stream = torch.cuda.current_stream(run.device)
    run.step(stream)
    torch.cuda.synchronize()
    run.check_status(stream)
    arrays = run.mesh.arrays()
    rp_exp, col_exp = expected_pattern(arrays)
    rows = sample_rows(run.mesh.n_elements, seed)
    tables = run.ref.tables()
    errs = []
    for params, out in zip(run.params, run.outputs()):
        assert np.array_equal(out.row_ptr.cpu().numpy(), rp_exp), "row_ptr differs"
        assert np.array_equal(out.col.cpu().numpy(), col_exp), "block columns differ"
        o = oracle.assemble(arrays, tables, run.spec.c, params, rows=rows)
        errs.append(compare_system(gather_rows_device(out, rows), o))
    return errs


@pytest.mark.parametrize("index", [1, 2, 3, 4, 5])
def test_bench_launch_full_size(oracle, index):
    """The default bench step of each config (config 2: the fused 3-method batch)."""
    run = workload.ConfigRun(index)
    if index == 2:
        assert run.batched
    _check_run(oracle, run, 2000 + index)


def test_bench_launch_repeated_steps_identical(oracle):
    """Config 4's persistent kernel run twice into the same buffers: bitwise identical (the
    bench times repeated steps; nothing may depend on leftover state)."""
    import torch
    run = workload.ConfigRun(4)
    stream = torch.cuda.current_stream(0)
    run.step(stream)
    torch.cuda.synchronize()
    first = run.outputs()[0].val.clone(), run.outputs()[0].rhs.clone()
    run.outputs()[0].val.fill_(float("nan"))
    run.step(stream)
    torch.cuda.synchronize()
    assert torch.equal(first[0], run.outputs()[0].val)
    assert torch.equal(first[1], run.outputs()[0].rhs)


def test_config2_single_assembly_path(oracle):
    """bench.py's single-assembly (--no-batch) figure for config 2: one bound launch per
    method."""
    run = workload.ConfigRun(2, batch=False)
    assert not run.batched
    _check_run(oracle, run, 2102)


def test_batched_c1_systems_equal_single_assembly(oracle):
    """bench.py --op c1-throughput: 512 copies of config 1 in one launch.  Every copy's system
    equals the single config-1 assembly bit for bit (offsets removed), and that one matches
    the oracle in full."""
    import torch
    single = workload.ConfigRun(1)
    stream = torch.cuda.current_stream(0)
    single.step(stream)
    batch = workload.BatchedSystemsRun(1, copies=512)
    batch.step(stream)
    torch.cuda.synchronize()
    batch.check_status(stream)
    s = single.outputs()[0]
    for b in (0, 1, 255, 511):
        sb = batch.system(b)
        for x, y in zip((s.row_ptr, s.col, s.val, s.rhs), (sb.row_ptr, sb.col, sb.val, sb.rhs)):
            assert torch.equal(x, y)
    o = oracle.assemble(single.mesh.arrays(), single.ref.tables(), single.spec.c, single.params[0])
    compare_system((s.row_ptr.cpu().numpy(), s.col.cpu().numpy(), s.val.cpu().numpy(),
                    s.rhs.cpu().numpy()), o)


def test_c1_graph_replay_equals_single_launch():
    """The CUDA-graph replay of config 1's launch (bench.py --op c1-throughput) writes the same
    bits as the eager launch."""
    import torch
    run = workload.ConfigRun(1)
    stream = torch.cuda.current_stream(0)
    run.step(stream)
    torch.cuda.synchronize()
    ref = [t.clone() for t in (run.outputs()[0].val, run.outputs()[0].rhs)]
    run.outputs()[0].val.fill_(0.0)
    g = workload.capture_graph(run, 4)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(ref[0], run.outputs()[0].val)
    assert torch.equal(ref[1], run.outputs()[0].rhs)
