"""A/B timing of the persistent annealing kernels (HOBO_SA_KERNEL=ring|stage|pair) on one config."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_19987_b200.hobo import HoboTensor  # noqa: E402
from workloads import cfg3_problem, uniform_colex  # noqa: E402

cfg = sys.argv[1]
if cfg == "cfg3":
    t, B = HoboTensor.from_problem(cfg3_problem()), 65536
elif cfg == "cfg4":
    t, B = HoboTensor.import_colex(4, 128, uniform_colex(4, 128, 4)), 262144
t0 = t.default_t_start() if cfg == "cfg3" else 5.0
t.sa_shard(1, 0, 128, 1, t0, t0)
kinds = sys.argv[2:] or ["ring", "stage", "pair"]
for kind in kinds:
    os.environ["HOBO_SA_KERNEL"] = kind
    t.set_profiling(True)
    t.sa_shard(2, 0, B, 1, t0, t0 / 10)
    ms = t.launch_stats()["kernel_ms"]
    X, E, _ = t.sa_shard(2, 0, B, 1, t0, t0 / 10)
    st = t.launch_stats()
    torch.cuda.synchronize()
    print(f"{cfg} {kind}: {st['kernel_ms']:.2f} ms/sweep, {B * t.N / (st['kernel_ms'] / 1e3) / 1e9:.3f} G flips/s, "
          f"{2 * st['mma_macs'] / (st['kernel_ms'] / 1e3) / 1e12:.0f} TF exec, mean E {E.double().mean().item():.2f}")
