"""SpMV experiment driver (tools only): times tools/libspmv_lab.so variants on config 4's
assembled matrix under L2 knobs (fetch granularity limit, persisting window on x)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from cuda.bindings import runtime as rt  # noqa: E402

from paper_1502_02941_b200 import workload  # noqa: E402

lab = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libspmv_lab.so"))
lab.lab_spmv.argtypes = [C.c_int, C.c_int, C.c_int] + [C.c_void_p] * 6
sp = workload.SpmvRun(4)
s = torch.cuda.current_stream()
sp.step(s)
torch.cuda.synchronize()
yref = sp.y.clone()
sysd = sp.system
n = sysd.row_ptr.numel() - 1
nbytes = sp.bytes_per_product()
err, maxp = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxPersistingL2CacheSize, 0)
err, maxw = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxAccessPolicyWindowSize, 0)
print(f"max persisting L2 {maxp / 2**20:.1f} MiB, max window {maxw / 2**20:.1f} MiB", flush=True)


def set_window(on: bool, frac_bytes: int = 0):
    v = rt.cudaStreamAttrValue()
    w = v.accessPolicyWindow
    if on:
        rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitPersistingL2CacheSize, maxp)
        w.base_ptr = sp.x.data_ptr()
        w.num_bytes = min(sp.x.numel() * 8, maxw)
        w.hitRatio = min(1.0, frac_bytes / w.num_bytes)
        w.hitProp = rt.cudaAccessProperty.cudaAccessPropertyPersisting
        w.missProp = rt.cudaAccessProperty.cudaAccessPropertyStreaming
    else:
        w.num_bytes = 0
        w.hitRatio = 0.0
        w.hitProp = rt.cudaAccessProperty.cudaAccessPropertyNormal
        w.missProp = rt.cudaAccessProperty.cudaAccessPropertyNormal
    err = rt.cudaStreamSetAttribute(s.cuda_stream, rt.cudaLaunchAttributeID.cudaLaunchAttributeAccessPolicyWindow, v)
    if not on:
        rt.cudaCtxResetPersistingL2Cache()
        rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitPersistingL2CacheSize, 0)
    return err


def run(variant, threads, gran=None, window=0):
    if gran is not None:
        rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitMaxL2FetchGranularity, gran)
    if window:
        set_window(True, window)
    y = torch.full_like(sp.y, float("nan"))
    args = [sysd.row_ptr.data_ptr(), sysd.col.data_ptr(), sysd.val.data_ptr(), sp.x.data_ptr(),
            y.data_ptr(), s.cuda_stream]
    per = lab.lab_spmv(variant, threads, n, *args)
    for _ in range(5):
        lab.lab_spmv(variant, threads, n, *args)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(30):
        lab.lab_spmv(variant, threads, n, *args)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 30
    ok = torch.equal(y, yref)
    if window:
        set_window(False)
    if gran is not None:
        rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitMaxL2FetchGranularity, 64)
    err, g = rt.cudaDeviceGetLimit(rt.cudaLimit.cudaLimitMaxL2FetchGranularity)
    print(f"v{variant} T={threads} gran={gran} window={window / 2**20:.0f}MiB ctas/sm={per}: "
          f"{ms:.4f} ms  {nbytes / ms / 1e6 / 6551:.3f} of roofline  equal={ok}", flush=True)


lab.lab_spmv_acc.argtypes = [C.c_int, C.c_int] + [C.c_void_p] * 5 + [C.c_int, C.c_void_p]


def split_parts(P):
    """column-split BSR parts: part p holds each row's blocks with col in [p N/P, (p+1) N/P)."""
    rp = sysd.row_ptr.long()
    counts = rp[1:] - rp[:-1]
    row_of = torch.repeat_interleave(torch.arange(n, device=rp.device), counts)
    colv = sysd.col.long()
    parts = []
    for p in range(P):
        lo, hi = p * n // P, (p + 1) * n // P
        m = (colv >= lo) & (colv < hi)
        c = torch.bincount(row_of[m], minlength=n)
        prp = torch.zeros(n + 1, dtype=torch.int32, device=rp.device)
        prp[1:] = torch.cumsum(c, 0).to(torch.int32)
        parts.append((prp, sysd.col[m].contiguous(), sysd.val[m].contiguous()))
    return parts


for P in (1, 2, 3, 4):
    parts = split_parts(P)
    y = torch.full_like(sp.y, float("nan"))

    def prod():
        for p, (prp, pc, pv) in enumerate(parts):
            lab.lab_spmv_acc(128, n, prp.data_ptr(), pc.data_ptr(), pv.data_ptr(), sp.x.data_ptr(),
                             y.data_ptr(), 1 if p else 0, s.cuda_stream)
    for _ in range(5):
        prod()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(30):
        prod()
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 30
    err = float(((y - yref).abs() / (yref.abs() + 1e-30)).max())
    print(f"column split P={P}: {ms:.4f} ms  {nbytes / ms / 1e6 / 6551:.3f} of roofline  max rel diff {err:.2e}", flush=True)
    del parts
