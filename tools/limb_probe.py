"""Energy / local-field kernel time at L = 2 and 3 bf16 limbs (binary x, 256-column tiles)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_19987_b200.hobo import HoboTensor  # noqa: E402
from workloads import int_twin_colex, uniform_colex  # noqa: E402

B = 65536
cases = {
    "o3n512_L2": lambda: HoboTensor.import_colex(3, 512, int_twin_colex(3, 512, 5, mod=1001, shift=500)),
    "o3n512_L3": lambda: HoboTensor.import_colex(3, 512, uniform_colex(3, 512, 6)),
    "o4n256_L3": lambda: HoboTensor.import_colex(4, 256, uniform_colex(4, 256, 7)),
}
for name in sys.argv[1:] or list(cases):
    t = cases[name]()
    g = torch.Generator().manual_seed(1)
    X = torch.randint(0, 2, (B, t.N), generator=g, dtype=torch.uint8).cuda()
    t.set_profiling(True)
    for what in ("energy", "field"):
        ms = []
        for _ in range(4):
            if what == "energy":
                t.energy(X)
            else:
                t.local_field(X)
            ms.append(t.launch_stats()["kernel_ms"])
        st = t.launch_stats()
        print(f"{name} {what}: {min(ms[1:]):.3f} ms, {2 * st['mma_macs'] / (min(ms[1:]) / 1e3) / 1e12:.0f} TF exec, "
              f"launches {st['launches']}")
