"""Per-call overhead of the energy + field call at a small batch (one GPU's share of cfg3 at 8
GPUs): wall time per synchronous call (with the argmin readback), per asynchronous call (no
best; a stream of calls, one sync at the end), and the Python binding alone."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2407_19987_b200 import HoboTensor  # noqa: E402
from workloads import cfg3_problem, x_bits  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
t = HoboTensor.from_problem(cfg3_problem())
Xd = torch.from_numpy(x_bits(3, B, 512)).cuda()
G = torch.empty(B, 512, device="cuda")
E = torch.empty(B, device="cuda")
s = torch.cuda.current_stream()
for _ in range(5):
    t.local_field(Xd, G, E, want_best=True, stream=s)
torch.cuda.synchronize()
n = 200
t0 = time.perf_counter()
for _ in range(n):
    t.local_field(Xd, G, E, want_best=True, stream=s)
sync_us = (time.perf_counter() - t0) / n * 1e6
t0 = time.perf_counter()
for _ in range(n):
    t.local_field(Xd, G, E, want_best=False, stream=s)
torch.cuda.synchronize()
async_us = (time.perf_counter() - t0) / n * 1e6
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record(s)
for _ in range(n):
    t.local_field(Xd, G, E, want_best=False, stream=s)
ev[1].record(s)
ev[1].synchronize()
dev_us = ev[0].elapsed_time(ev[1]) / n * 1e3
print(f"B={B}: synchronous call {sync_us:.1f} us, asynchronous stream {async_us:.1f} us/call, device {dev_us:.1f} us/call")
