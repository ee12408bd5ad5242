"""Per-warp timing of the persistent P1 kernel on config 4 (tuning build, dgb_tuning_set_diag):
effective SM clock inside the kernel, spread of the warps' finishing times, chunks per SM."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1502_02941_b200 import capi, workload  # noqa: E402

lib = capi.load()
stream = torch.cuda.current_stream()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
run = workload.ConfigRun(int(os.environ.get("CFG", "4")))
n_warps = 148 * 12
diag = torch.zeros(4 * n_warps, dtype=torch.int64, device="cuda")
lib.dgb_tuning_set_diag.argtypes = [C.c_void_p, C.c_void_p]
assert lib.dgb_tuning_set_diag(run.plan._h, C.c_void_p(diag.data_ptr())) == 0
for rep in range(6):
    flush.fill_(float(rep))
    run.step(stream)
    torch.cuda.synchronize()
    d = diag.cpu().numpy().reshape(n_warps, 4)
    t0, t1, cyc = d[:, 0], d[:, 1], d[:, 2]
    smid = d[:, 3] & 0xFFFFFFFF
    chunks = d[:, 3] >> 32
    start = t0.min()
    dur = (t1 - t0).astype(np.float64)
    mhz = cyc / dur * 1e3
    end = (t1 - start) / 1e3
    beg = (t0 - start) / 1e3
    per_sm = np.array([chunks[smid == s].sum() for s in np.unique(smid)])
    print(f"rep {rep}: kernel span {end.max():.1f} us; warp start max {beg.max():.1f} us; "
          f"warp end min/median/max {end.min():.1f}/{np.median(end):.1f}/{end.max():.1f} us; "
          f"SM clock MHz min/median/max {mhz.min():.0f}/{np.median(mhz):.0f}/{mhz.max():.0f}; "
          f"chunks per warp min/max {chunks.min()}/{chunks.max()}; per SM min/max {per_sm.min()}/{per_sm.max()}",
          flush=True)
sm_end = np.array([end[smid == s].max() for s in np.unique(smid)])
print("per-SM last end (us), sorted:", np.round(np.sort(sm_end), 1).tolist())
