"""The multilinear field (gradient descent's contraction at real p) on cfg3, 65,536 candidates."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_19987_b200.hobo import HoboTensor  # noqa: E402
from workloads import cfg3_problem, h  # noqa: E402

B = 65536
t = HoboTensor.from_problem(cfg3_problem())
u = ((h(3, 3, np.arange(B, dtype=np.uint64)[:, None], np.arange(t.N, dtype=np.uint64)[None, :]) >> np.uint64(40))
     .astype(np.float32) * np.float32(2.0 ** -24))
P = torch.from_numpy(u).cuda().to(torch.bfloat16).contiguous()
G = torch.empty(B, t.N, device="cuda")
E = torch.empty(B, device="cuda")
t.set_profiling(True)
for _ in range(3):
    t.multilinear_field(P, G, E)
    print("kernel ms", t.launch_stats()["kernel_ms"])
torch.cuda.synchronize()
