import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2407_19987_b200.hobo import HoboTensor
from workloads import uniform_colex
t = HoboTensor.import_colex(4, 128, uniform_colex(4, 128, 4))
t.sa_shard(1, 0, 128, 1, 5.0, 5.0)
t.set_profiling(True)
for nb in (148, 74, 37, 10):
    B = nb * 128
    t.sa_shard(2, 0, B, 1, 5.0, 0.5)
    ms = t.launch_stats()["kernel_ms"]
    print(f"{nb} blocks: {ms:.2f} ms/sweep = {ms * 1e3 / 128:.1f} us/site")
