import sys, time
sys.path.insert(0, '.')
import torch
from paper_1502_02941_b200 import workload
sp = workload.SpmvRun(4)
s = torch.cuda.current_stream()
torch.cuda.synchronize()
for rnd in range(3):
    t0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(20):
        sp.step(s)
    e1.record(s)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"round {rnd}: host enqueue {1e3*(t1-t0)/20:.3f} ms/call, device {e0.elapsed_time(e1)/20:.3f} ms/product, wall {1e3*(t2-t0)/20:.3f}", flush=True)
