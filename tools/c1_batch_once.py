"""One launch of the 512-system config-1 batch (for an ncu capture of exactly that launch)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1502_02941_b200 import workload  # noqa: E402

run = workload.BatchedSystemsRun(1, int(os.environ.get("COPIES", "512")))
stream = torch.cuda.current_stream()
for _ in range(3):
    run.step(stream)
torch.cuda.synchronize()
