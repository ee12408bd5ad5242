"""Batch (fused / unfused) vs single assemblies, warp-specialised or not: max differences."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_1502_02941_b200 import capi, dgfem, problems, shard

cfg = problems.CONFIGS[2]
mesh = dgfem.unit_square_mesh(48)
ref = dgfem.ReferenceElement(cfg.degree, cfg.quad_order)
spec = problems.config_problem(2, mesh.n_elements)
methods = [capi.SIPG, capi.NIPG, capi.IIPG]
params = [dgfem.config_parameters(cfg, m) for m in methods]


def run(fuse, ws, batch):
    a = [shard.ShardAssembler(mesh, ref, spec, 0, 0, mesh.n_elements, bind=True)]
    a += [shard.ShardAssembler(mesh, ref, spec, 0, 0, mesh.n_elements, share=a[0]) for _ in methods[1:]]
    a[0].plan.set_option(capi.OPTION_BATCH_FUSE, fuse)
    a[0].plan.set_option(capi.OPTION_WARP_SPECIALIZED, ws)
    if batch:
        shard.assemble_batch(a, params)
    else:
        for x, p in zip(a, params):
            x.assemble(p)
    return [[t.cpu().numpy() for t in (x.out.row_ptr, x.out.col, x.out.val, x.out.rhs)] for x in a]


ref_out = run(0, 0, False)
for fuse, ws, batch in [(0, 1, False), (0, 0, True), (1, 0, True), (1, 1, True), (0, 1, True)]:
    o = run(fuse, ws, batch)
    msg = []
    for m in range(3):
        for nm, x, y in zip(["rp", "col", "val", "rhs"], o[m], ref_out[m]):
            d = np.abs(x.astype(float) - y.astype(float)).max()
            msg.append(f"{nm}{m}={d:.1e}")
    print(f"fuse={fuse} ws={ws} batch={batch}: " + " ".join(msg))
