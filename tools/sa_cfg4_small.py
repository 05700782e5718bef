"""cfg4 annealing on 10 chain blocks, one sweep (short, for ncu captures of the site pipeline)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_19987_b200.hobo import HoboTensor  # noqa: E402
from workloads import uniform_colex  # noqa: E402

t = HoboTensor.import_colex(4, 128, uniform_colex(4, 128, 4))
t.sa_shard(2, 0, 1280, 1, 5.0, 0.5)
torch.cuda.synchronize()
