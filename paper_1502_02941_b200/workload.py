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
