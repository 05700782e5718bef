import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2407_19987_b200 import hobo as H
from workloads import x_bits, cfg3_problem
from workloads.gen import int_encoded_problem
for name, p, B in (("cfg3 N=512", cfg3_problem(), 65536), ("intenc N=1024", int_encoded_problem(256, 4, 2048, 4096, 7), 65536)):
    t = H.HoboTensor.from_problem(p)
    X = torch.from_numpy(x_bits(3, B, p.N)).cuda()
    t.local_field(X); torch.cuda.synchronize()
    t.set_profiling(True)
    ks = []
    for _ in range(5):
        t.local_field(X); torch.cuda.synchronize()
        ks.append(t.launch_stats()["kernel_ms"])
    st = t.launch_stats()
    ms = sorted(ks)[2]
    hw = 2 * 8192 * 148 * 1.965e9
    print(name, "kind", st["i8_planes"], "kernel ms", round(ms, 3), "exec frac", round(2 * st["mma_macs"] / (ms / 1e3) / hw, 3))
