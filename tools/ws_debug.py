"""Warp-specialised vs monolithic kernel: max differences per output (debug aid)."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_1502_02941_b200 import capi, dgfem, problems, shard

deg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 48
cfg = problems.CONFIGS[2]
mesh = dgfem.unit_square_mesh(n)
ref = dgfem.ReferenceElement(deg, 2 * deg)
spec = problems.config_problem(2, mesh.n_elements)
p = dgfem.config_parameters(cfg, capi.SIPG)
res = {}
for ws in (1, 0):
    a = shard.ShardAssembler(mesh, ref, spec, 0, 0, mesh.n_elements, bind=True)
    a.plan.set_option(capi.OPTION_WARP_SPECIALIZED, ws)
    o = a.assemble(p)
    res[ws] = [x.cpu().numpy() for x in (o.row_ptr, o.col, o.val, o.rhs)]
names = ["row_ptr", "col", "val", "rhs"]
nl = ref.n_local
for nm, x, y in zip(names, res[1], res[0]):
    d = np.abs(x.astype(float) - y.astype(float))
    i = int(d.argmax())
    print(nm, "max diff", d.max(), "at", i, "n_diff", int((d > 0).sum()), "of", d.size,
          "vals", x.flat[i], y.flat[i])
    if nm == "val" and d.max() > 0:
        blk = i // (nl * nl)
        rows = np.searchsorted(res[0][0], blk, side="right") - 1
        print("  block", blk, "row", rows, "col", res[0][1][blk], "entry", i % (nl * nl))
        bad = np.unique(np.nonzero(d > 1e-12 * np.abs(y).max())[0] // (nl * nl))
        print("  bad blocks", bad[:20], len(bad))
