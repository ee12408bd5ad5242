"""Element-row sharding of the assembly across ranks.

Block rows are independent in the gather formulation, so rank r assembles rows
[begin_r, end_r) of the global K and F with no collective on the data path.  The only
exchange is bookkeeping: each shard's block count, whose exclusive prefix over ranks is the
shard's offset in the global BSR (global row_ptr = shard row_ptr + offset), and the global
InflowOnNeumann detail (the minimum offending edge over ranks, as the reference reports the
lowest one).  Row ranges split like the reference's run_chunks (assembly.cpp:38-39).
"""
from __future__ import annotations

import ctypes as C

from . import capi


def row_range(n_rows: int, rank: int, world: int) -> tuple[int, int]:
    """[begin, end) of rank `rank` (contiguous, balanced; assembly.cpp:38-39 arithmetic)."""
    return rank * n_rows // world, (rank + 1) * n_rows // world


def block_count(mesh_view, begin: int, end: int) -> int:
    """BSR blocks of rows [begin, end) of a host mesh (dgb_count_blocks_host)."""
    n = capi.load().dgb_count_blocks_host(C.byref(mesh_view), begin, end)
    if n < 0:
        raise ValueError("bad row range")
    return int(n)


def global_block_offset(local_blocks: int, group=None) -> tuple[int, int]:
    """(offset of this shard's first block, total blocks) via one all_gather of counts."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    mine = torch.tensor([local_blocks], dtype=torch.int64, device=dev)
    allc = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(allc, mine, group=group)
    counts = [int(t.item()) for t in allc]
    r = dist.get_rank(group)
    return sum(counts[:r]), sum(counts)


def global_error_edge(local_edge: int, group=None) -> int:
    """Lowest InflowOnNeumann edge over all shards (-1 when none)."""
    import torch
    import torch.distributed as dist
    big = 2**62
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([local_edge if local_edge >= 0 else big], dtype=torch.int64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    v = int(t.item())
    return -1 if v == big else v


class ShardAssembler:
    """GPU assembly of one rank's block rows (full mesh replicated in HBM, ~46 B/element)."""

    def __init__(self, mesh, ref, problem, device: int, begin: int, end: int, share=None,
                 bind: bool = False):
        """share: another ShardAssembler whose plan and device copies to reuse; bind: compute
        the shard's BSR pattern once (dgb_plan_bind_mesh), one kernel per assembly after."""
        from . import dgfem
        self.begin, self.end = begin, end
        if share is not None:
            self.plan, self.dmesh, self.dprob = share.plan, share.dmesh, share.dprob
        else:
            self.plan = dgfem.Plan(ref.view, device)
            self.dmesh = dgfem.DeviceMesh(mesh, device)
            self.dprob = dgfem.DeviceProblem(problem, device)
        self.n_blocks = block_count(mesh.view, begin, end)
        if bind:
            self.plan.bind_mesh(self.dmesh, begin, end)
        import torch
        dev = torch.device("cuda", device)
        nl = ref.n_local
        self.out = dgfem.BsrSystem(torch.empty(end - begin + 1, dtype=torch.int32, device=dev),
                                   torch.empty(self.n_blocks, dtype=torch.int32, device=dev),
                                   torch.empty((self.n_blocks, nl, nl), dtype=torch.float64, device=dev),
                                   torch.empty((end - begin, nl), dtype=torch.float64, device=dev), nl)

    def assemble(self, params, stream=None, check: bool = True):
        import torch
        from . import dgfem
        lib = capi.load()
        if stream is None:
            stream = torch.cuda.current_stream(self.plan.device)
        h = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        b = self.out.struct()
        dgfem._check(lib.dgb_assemble_rows(self.plan._h, C.byref(self.dmesh.view),
                                           C.byref(self.dprob.c), C.byref(params), self.begin,
                                           self.end, C.byref(b), self.out.rhs.data_ptr(),
                                           C.c_void_p(h)))
        if check:
            dgfem._check(lib.dgb_plan_status(self.plan._h, C.c_void_p(h)))
        return self.out


def assemble_batch(assemblers, params_list, stream=None, check: bool = True):
    """dgb_assemble_batch over ShardAssemblers sharing one plan, device mesh and row range
    (one launch for all parameter sets when the rows are bound)."""
    import torch
    from . import dgfem
    lib = capi.load()
    a0 = assemblers[0]
    if stream is None:
        stream = torch.cuda.current_stream(a0.plan.device)
    h = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
    n = len(assemblers)
    outs = (capi.Bsr * n)(*[a.out.struct() for a in assemblers])
    rhs = (C.c_void_p * n)(*[a.out.rhs.data_ptr() for a in assemblers])
    prm = (capi.Params * n)(*params_list)
    dgfem._check(lib.dgb_assemble_batch(a0.plan._h, C.byref(a0.dmesh.view), C.byref(a0.dprob.c),
                                        prm, n, a0.begin, a0.end, outs, rhs, C.c_void_p(h)))
    if check:
        dgfem._check(lib.dgb_plan_status(a0.plan._h, C.c_void_p(h)))
    return [a.out for a in assemblers]
