"""TT-form energies of the paper's TSP tensor over 4M random candidates (for ncu captures)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_19987_b200.hobo import HoboTensor  # noqa: E402
from workloads import tsp, x_bits  # noqa: E402

t = HoboTensor.from_problem(tsp())
print("ranks", t.tt_build(0.0))
B = 1 << 22
X = torch.from_numpy(x_bits(11, B, t.N)).cuda()
for _ in range(3):
    E, best = t.tt_energy(X)
torch.cuda.synchronize()
print("best", best)
