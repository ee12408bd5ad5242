"""The launch sequence behind every number `bench.py` reports for a BASELINE.json config, in one
place, so that the full-size parity tests (tests/test_gpu_bench_paths.py) run exactly the
launches the bench times.

A `ConfigRun` holds one config's device-resident mesh, coefficients, plan and outputs:

* one `ShardAssembler` per method (shared plan and device mesh), rows [begin, end) of the global
  mesh (`world` config-sized squares side by side for weak scaling);
* the pattern bound once (`dgb_plan_bind_mesh`: count + scan + adjacency), its device time
  recorded in `bind_ms`;
* `step()`: one `dgb_assemble_batch` for a multi-method config (config 2: the fused,
  warp-specialised launch), otherwise one `dgb_assemble_rows` per method -- the reference's
  `assemble_all` + `stiffness()` (assembly.cpp:725-737, assembly.cpp:508) per method.
"""
from __future__ import annotations

import ctypes as C

from . import capi, dgfem, problems, shard


class ConfigRun:
    def __init__(self, index: int, device: int = 0, rank: int = 0, world: int = 1,
                 batch: bool = True, bind: bool = True, methods=None, options: dict | None = None,
                 mesh=None):
        """options: plan options by capi.OPTION_* value (tuning runs only; the defaults are the
        bench's).  methods: override the config's method list (e.g. a single method)."""
        import torch
        self.index, self.device, self.world = index, device, world
        self.cfg = cfg = problems.CONFIGS[index]
        self.mesh = mesh if mesh is not None else dgfem.config_mesh(cfg, strips=world)
        self.ref = dgfem.ReferenceElement(cfg.degree, cfg.quad_order)
        self.spec = problems.config_problem(index, self.mesh.n_elements)
        self.methods = tuple(cfg.methods if methods is None else methods)
        self.params = [dgfem.config_parameters(cfg, m) for m in self.methods]
        self.begin, self.end = shard.row_range(self.mesh.n_elements, rank, world)
        first = shard.ShardAssembler(self.mesh, self.ref, self.spec, device, self.begin, self.end)
        self.plan = first.plan
        for opt, value in (options or {}).items():
            if value is not None:
                self.plan.set_option(opt, value)
        self.bound = bind
        self.bind_ms = None
        if bind:
            stream = torch.cuda.current_stream(device)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            torch.cuda.synchronize(device)
            ev[0].record(stream)
            self.plan.bind_mesh(first.dmesh, self.begin, self.end, stream=stream)
            ev[1].record(stream)
            torch.cuda.synchronize(device)
            self.bind_ms = ev[0].elapsed_time(ev[1])
        self.shards = [first] + [shard.ShardAssembler(self.mesh, self.ref, self.spec, device,
                                                      self.begin, self.end, share=first)
                                 for _ in self.params[1:]]
        self.batched = batch and len(self.params) > 1

    @property
    def n_rows(self) -> int:
        return self.end - self.begin

    def step(self, stream, kernel_events=None, check: bool = False) -> None:
        """One step: every method's assembly of the rows.  kernel_events: per launch, a
        (start, end) torch event pair the plan records around its block-row kernel on `stream`
        (dgb_plan_set_kernel_events); a batched step uses the first pair only."""
        lib = capi.load()
        h = self.plan._h
        if self.batched:
            if kernel_events is not None:
                ks, ke = kernel_events[0]
                lib.dgb_plan_set_kernel_events(h, C.c_void_p(ks.cuda_event), C.c_void_p(ke.cuda_event))
            shard.assemble_batch(self.shards, self.params, stream=stream, check=check)
        else:
            for i, (p, sh) in enumerate(zip(self.params, self.shards)):
                if kernel_events is not None:
                    ks, ke = kernel_events[i]
                    lib.dgb_plan_set_kernel_events(h, C.c_void_p(ks.cuda_event), C.c_void_p(ke.cuda_event))
                sh.assemble(p, stream=stream, check=check)
        lib.dgb_plan_set_kernel_events(h, None, None)

    def launches_per_step(self) -> int:
        return 1 if self.batched else len(self.params)

    def check_status(self, stream) -> None:
        dgfem._check(capi.load().dgb_plan_status(self.plan._h, C.c_void_p(stream.cuda_stream)))

    def outputs(self):
        """[BsrSystem] per method, rows [begin, end) (device tensors)."""
        return [sh.out for sh in self.shards]


class SpmvRun:
    """Config 4's A*x check (BASELINE.json configs[3]: "100 BSR SpMVs on seeded uniform[-1,1]
    x"): K assembled once by the bench's own launch (ConfigRun), then `step()` = one product
    y = K x through dgb_spmv (the reference's matvec, sparse.cpp:116-129)."""

    def __init__(self, index: int = 4, device: int = 0):
        import torch
        self.run = ConfigRun(index, device)
        stream = torch.cuda.current_stream(device)
        self.run.step(stream, check=True)
        self.system = self.run.outputs()[0]
        n = self.run.n_rows * self.run.ref.n_local
        self.x = torch.from_numpy(2.0 * problems.uniform01(problems.SEED_SPMV_X, n) - 1.0).to(
            torch.device("cuda", device))
        self.y = torch.empty_like(self.x)
        self.device = device
        self._b = self.system.struct()

    def step(self, stream, y=None) -> None:
        out = self.y if y is None else y
        dgfem._check(capi.load().dgb_spmv(C.byref(self._b), self.x.data_ptr(), out.data_ptr(),
                                          C.c_void_p(stream.cuda_stream)))

    def bytes_per_product(self) -> int:
        """8 nl^2 nnzb + 4 nnzb + 4 (E + 1) + 16 nl E (values, block columns,
        row pointer, x read once, y written once)."""
        nl, E = self.run.ref.n_local, self.run.n_rows
        nnzb = self.system.col.shape[0]
        return 8 * nl * nl * nnzb + 4 * nnzb + 4 * (E + 1) + 16 * nl * E


def replicated_raw(raw: dict, copies: int) -> dict:
    """The disjoint union of `copies` copies of a raw mesh (nodes, elements, boundary pairs):
    copy b's node and element indices are offset by b n_nodes and b n_elements, so no edge is
    shared between copies and the assembled union is block diagonal -- copy b's system is block
    rows [b E, (b+1) E) with block columns offset by b E."""
    import numpy as np
    nn = raw["nodes"].shape[0]
    off = (np.arange(copies, dtype=np.int64) * nn)[:, None, None]
    rep = lambda a: (a[None].astype(np.int64) + off).reshape(-1, a.shape[1]).astype(np.int32)  # noqa: E731
    return {"nodes": np.tile(raw["nodes"], (copies, 1)), "elements": rep(raw["elements"]),
            "dirichlet": rep(raw["dirichlet"]), "neumann": rep(raw["neumann"])}


class BatchedSystemsRun(ConfigRun):
    """`copies` independent systems of config `index` in ONE launch: the bound block-row kernel
    over the disjoint union of the config's mesh repeated `copies` times (BASELINE.md §2 note 1:
    a small config's throughput figure).  System b is block rows [b E, (b+1) E) of the output,
    its block columns offset by b E and its row_ptr by b nnzb; `system(b)` returns it with both
    offsets removed (the reference's per-call DgSystem of that copy)."""

    def __init__(self, index: int = 1, copies: int = 512, device: int = 0, options: dict | None = None):
        cfg = problems.CONFIGS[index]
        single = dgfem.config_mesh(cfg)
        self.copies, self.E_sys = copies, single.n_elements
        self.nnzb_sys = single.n_elements + 2 * single.n_interior_edges
        r = replicated_raw(single.raw(), copies)
        union = dgfem.build_mesh(r["nodes"], r["elements"], r["dirichlet"], r["neumann"])
        super().__init__(index, device, mesh=union, options=options)

    def system(self, b: int):
        out = self.outputs()[0]
        E, nb = self.E_sys, self.nnzb_sys
        rp = out.row_ptr[b * E:(b + 1) * E + 1] - b * nb
        return dgfem.BsrSystem(rp, out.col[b * nb:(b + 1) * nb] - b * E,
                               out.val[b * nb:(b + 1) * nb], out.rhs[b * E:(b + 1) * E],
                               out.block_dim)


def capture_graph(run: ConfigRun, n: int):
    """A CUDA graph of `n` consecutive steps of `run` (its launches captured on a side stream;
    replay() re-issues them with one launch call).  The plan must already be bound."""
    import torch
    side = torch.cuda.Stream(run.device)
    side.wait_stream(torch.cuda.current_stream(run.device))
    with torch.cuda.stream(side):
        run.step(side)          # warm (first-launch attribute setup happens outside capture)
    torch.cuda.current_stream(run.device).wait_stream(side)
    torch.cuda.synchronize(run.device)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        for _ in range(n):
            run.step(side)
    return g
