"""Probe of the annealing sweep on cfg3 (65,536 chains): per-site time, for ncu captures."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2407_19987_b200.hobo import HoboTensor  # noqa: E402
from workloads import cfg3_problem  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
t = HoboTensor.from_problem(cfg3_problem())
t0 = t.default_t_start()
t.sa_shard(1, 0, 128, 0, t0, t0)          # device init
torch.cuda.synchronize()
w = time.time()
t.sa_shard(1, 0, 128, 1, t0, t0)          # builds the site layouts
torch.cuda.synchronize()
print("site-layout build s", time.time() - w)
t.sa_shard(1, 0, B, 1, t0, t0)
torch.cuda.synchronize()
t.set_profiling(True)
for ta, tb in ((t0, t0 / 10), (t0 / 1000, t0 / 10000)):
    X, E, Et = t.sa_shard(2, 0, B, sweeps, ta, tb)
    st = t.launch_stats()
    print(f"T {ta:.4g}->{tb:.4g}: {st['kernel_ms']:.2f} ms, {st['kernel_ms'] * 1e3 / (sweeps * t.N):.1f} us/site,"
          f" mean E {E.double().mean().item():.1f}")
