"""CPU, world_size 2 over gloo: the sharded path's host logic (row ranges, the block-count
exchange that gives each shard its global offset, the global InflowOnNeumann reduction).  Each
rank assembles its shard with the C restatement (no GPU here); the concatenation of shards
must equal the full assembly bitwise."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, result_dir):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist

    from oracle.oracle import OracleLib
    from paper_1502_02941_b200 import dgfem, problems, shard
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    cfg = problems.CONFIGS[3]
    mesh = dgfem.unit_square_mesh(9, cfg.jitter, problems.SEED_JITTER, False, 0, cfg.neumann_sides)
    ref = dgfem.ReferenceElement(cfg.degree, cfg.quad_order)
    spec = problems.config_problem(3)
    params = dgfem.config_parameters(cfg, cfg.methods[0])
    b, e = shard.row_range(mesh.n_elements, rank, world)
    nblk = shard.block_count(mesh.view, b, e)
    off, total = shard.global_block_offset(nblk)
    rp, col, val, rhs = OracleLib().assemble(mesh.arrays(), ref.tables(), spec.c, params,
                                             rows=np.arange(b, e, dtype=np.int32), threads=1)
    assert rp[-1] == nblk
    err = shard.global_error_edge(7 if rank == 1 else -1)
    none = shard.global_error_edge(-1)
    np.savez(os.path.join(result_dir, f"rank{rank}.npz"), begin=b, end=e, off=off, total=total,
             rp=rp + off, col=col, val=val, rhs=rhs, err=err, none=none)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_shards_concatenate_to_full_assembly(tmp_path):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    from oracle.oracle import OracleLib
    from paper_1502_02941_b200 import dgfem, problems
    cfg = problems.CONFIGS[3]
    mesh = dgfem.unit_square_mesh(9, cfg.jitter, problems.SEED_JITTER, False, 0, cfg.neumann_sides)
    ref = dgfem.ReferenceElement(cfg.degree, cfg.quad_order)
    full = OracleLib().assemble(mesh.arrays(), ref.tables(), problems.config_problem(3).c,
                                dgfem.config_parameters(cfg, cfg.methods[0]), threads=1)
    parts = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    assert parts[0]["begin"] == 0 and parts[-1]["end"] == mesh.n_elements
    assert parts[0]["end"] == parts[1]["begin"]
    assert all(int(p["total"]) == full[0][-1] for p in parts)
    rp = np.concatenate([parts[0]["rp"][:-1], parts[1]["rp"]])
    np.testing.assert_array_equal(rp, full[0])
    np.testing.assert_array_equal(np.concatenate([p["col"] for p in parts]), full[1])
    np.testing.assert_array_equal(np.concatenate([p["val"] for p in parts]), full[2])
    np.testing.assert_array_equal(np.concatenate([p["rhs"] for p in parts]), full[3])
    assert all(int(p["err"]) == 7 and int(p["none"]) == -1 for p in parts)


def test_row_ranges_partition():
    from paper_1502_02941_b200 import shard
    for n in (1, 7, 131072):
        for w in (1, 2, 3, 8):
            ranges = [shard.row_range(n, r, w) for r in range(w)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))


def _spmv_worker(rank, world, port, result_dir):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch
    import torch.distributed as dist

    from oracle.oracle import OracleLib
    from paper_1502_02941_b200 import dgfem, problems, shard
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    cfg = problems.CONFIGS[4]
    mesh = dgfem.unit_square_mesh(12, 0.0, 0, True, problems.SEED_PERMUTE, 0)   # permuted
    ref = dgfem.ReferenceElement(cfg.degree, cfg.quad_order)
    spec = problems.config_problem(4)
    params = dgfem.config_parameters(cfg, cfg.methods[0])
    b, e = shard.row_range(mesh.n_elements, rank, world)
    orc = OracleLib()
    rp, col, val, _ = orc.assemble(mesh.arrays(), ref.tables(), spec.c, params,
                                   rows=np.arange(b, e, dtype=np.int32), threads=1)
    nl = ref.n_local
    x = 2.0 * problems.uniform01(problems.SEED_SPMV_X, mesh.n_elements * nl) - 1.0

    def cpu_spmv(row_ptr, col_local, v, x_ext, y):
        y[:] = torch.from_numpy(orc.spmv(row_ptr, col_local.numpy(), v, x_ext.numpy(), threads=1))

    h = shard.HaloSpmv(rp, torch.from_numpy(col), nl, mesh.n_elements, b, e, local_spmv=cpu_spmv)
    y = torch.zeros((e - b) * nl, dtype=torch.float64)
    h(val, torch.from_numpy(x[b * nl:e * nl].copy()), y)
    np.savez(os.path.join(result_dir, f"spmv{rank}.npz"), y=y.numpy(), halo=h.n_halo,
             sent=sum(h.send_counts))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world", [2, 3])
def test_halo_spmv_equals_full_product(tmp_path, world):
    """The sharded SpMV (halo exchange of x over torch.distributed) concatenates to the full
    product of the C restatement, bitwise (same per-row summation order)."""
    mp.start_processes(_spmv_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    from oracle.oracle import OracleLib
    from paper_1502_02941_b200 import dgfem, problems
    cfg = problems.CONFIGS[4]
    mesh = dgfem.unit_square_mesh(12, 0.0, 0, True, problems.SEED_PERMUTE, 0)
    ref = dgfem.ReferenceElement(cfg.degree, cfg.quad_order)
    orc = OracleLib()
    rp, col, val, _ = orc.assemble(mesh.arrays(), ref.tables(), problems.config_problem(4).c,
                                   dgfem.config_parameters(cfg, cfg.methods[0]))
    x = 2.0 * problems.uniform01(problems.SEED_SPMV_X, mesh.n_elements * ref.n_local) - 1.0
    full = orc.spmv(rp, col, val, x, threads=1)
    parts = [np.load(os.path.join(tmp_path, f"spmv{r}.npz")) for r in range(world)]
    np.testing.assert_array_equal(np.concatenate([p["y"] for p in parts]), full)
    assert all(int(p["halo"]) > 0 for p in parts)            # permuted mesh: real halos
    assert sum(int(p["halo"]) for p in parts) == sum(int(p["sent"]) for p in parts)
