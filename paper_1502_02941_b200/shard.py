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


class HaloSpmv:
    """y = K x for a row-sharded BSR: rank r owns block rows [begin, end)
    of K and the matching slice of x; a product needs x at the shard's off-shard block columns
    (the 1-ring halo).  Built once per shard:

      * the halo plan: the remote block columns, grouped by owning rank (row_range), and --
        after one exchange of request lists -- what this rank sends to every peer;
      * a column map: global block column -> index in [owned x | halo x].

    Per product: one variable-size all_to_all of nl-blocks of x (NCCL over NVLink on the GPU,
    gloo in the CPU tests), then the local BSR product on [owned | halo] with the remapped
    columns.  `local_spmv(x_ext, y)` is dgb_spmv on the GPU (default) or any callable with
    the same meaning (the tests pass the C restatement's CPU product)."""

    def __init__(self, row_ptr, col, block_dim: int, n_rows_global: int, begin: int, end: int,
                 group=None, local_spmv=None):
        import numpy as np
        import torch
        import torch.distributed as dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.nl, self.begin, self.end = block_dim, begin, end
        self.n_own = end - begin
        col_h = col.cpu().numpy() if hasattr(col, "cpu") else np.asarray(col)
        ranges = [row_range(n_rows_global, r, self.world) for r in range(self.world)]
        owner = np.zeros(0, np.int64)
        remote = np.unique(col_h[(col_h < begin) | (col_h >= end)])
        if remote.size:
            starts = np.array([b for b, _ in ranges])
            owner = np.searchsorted(starts, remote, side="right") - 1
        self.recv_cols = [remote[owner == p] for p in range(self.world)]   # sorted per peer
        # exchange request lists: counts, then the block ids each peer wants from this rank
        dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
        cnt = torch.tensor([len(c) for c in self.recv_cols], dtype=torch.int64, device=dev)
        cnt_in = torch.empty_like(cnt)
        dist.all_to_all_single(cnt_in, cnt, group=group)
        self.recv_counts = [int(v) for v in cnt.tolist()]
        self.send_counts = [int(v) for v in cnt_in.tolist()]
        req = torch.from_numpy(np.concatenate(self.recv_cols).astype(np.int64) if remote.size
                               else np.zeros(0, np.int64)).to(dev)
        want = torch.empty(sum(self.send_counts), dtype=torch.int64, device=dev)
        dist.all_to_all_single(want, req, self.send_counts, self.recv_counts, group=group)
        self.send_local = (want - begin).to(torch.int64)                  # owned block indices
        # column map: owned -> [0, n_own), halo (peer order, sorted) -> n_own + position
        halo_pos = {int(c): self.n_own + i for i, c in enumerate(np.concatenate(self.recv_cols))} \
            if remote.size else {}
        remap = np.where((col_h >= begin) & (col_h < end), col_h - begin, -1)
        for i in np.nonzero(remap < 0)[0]:
            remap[i] = halo_pos[int(col_h[i])]
        self.col_local = torch.from_numpy(remap.astype(np.int32)).to(col.device if hasattr(col, "device") else "cpu")
        self.row_ptr = row_ptr
        self.n_halo = len(halo_pos)
        self.local_spmv = local_spmv

    def exchange(self, x_own):
        """[owned | halo] blocks of x for this rank (x_own: [n_own * nl])."""
        import torch
        import torch.distributed as dist
        nl = self.nl
        xb = x_own.reshape(self.n_own, nl)
        send = xb.index_select(0, self.send_local.to(xb.device)).reshape(-1).contiguous()
        recv = torch.empty(self.n_halo * nl, dtype=x_own.dtype, device=x_own.device)
        dist.all_to_all_single(recv, send, [c * nl for c in self.recv_counts],
                               [c * nl for c in self.send_counts], group=self.group)
        return torch.cat([x_own, recv])

    def __call__(self, val, x_own, y_own):
        x_ext = self.exchange(x_own)
        if self.local_spmv is not None:
            self.local_spmv(self.row_ptr, self.col_local, val, x_ext, y_own)
        else:  # dgb_spmv on the device
            from . import dgfem
            import torch
            b = capi.Bsr()
            b.n_block_rows, b.block_dim, b.nnzb = self.n_own, self.nl, self.col_local.numel()
            b.row_ptr, b.col, b.val = self.row_ptr.data_ptr(), self.col_local.data_ptr(), val.data_ptr()
            stream = torch.cuda.current_stream(x_own.device)
            dgfem._check(capi.load().dgb_spmv(C.byref(b), x_ext.data_ptr(), y_own.data_ptr(),
                                              C.c_void_p(stream.cuda_stream)))
        return y_own
