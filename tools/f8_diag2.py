"""e4m3 vs bf16 on two-bit candidates of the last K-block pair, by batch size / split."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_19987_b200 import hobo as H
exec(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "f8_diag.py")).read().split("def run(")[0].split("from workloads.gen import canonical_cells_all")[1])
from workloads import h, x_bits
from workloads.gen import canonical_cells_all
N = 128
idx, val = pow2_int_cells(3, N, 5)
deg = (idx[:, 0] != idx[:, 1]).astype(int) + (idx[:, 1] != idx[:, 2]).astype(int) + 1
ii, vv = idx[deg == 3], val[deg == 3]
t = H.HoboTensor.import_cells(3, N, ii, vv)
os.environ["HOBO_F8"] = "0"
tb = H.HoboTensor.import_cells(3, N, ii, vv)
del os.environ["HOBO_F8"]
for B in (64, 496, 8192, 20000):
    X = np.zeros((B, N), np.uint8)
    for r in range(B):
        a = 63 + (r % 64)
        X[r, a] = 1
        X[r, 127] = 1
    Xd = torch.from_numpy(X).cuda()
    for pair in ("0", "1"):
        os.environ["HOBO_PAIR"] = pair
        G, E = t.local_field(Xd)
        os.environ["HOBO_F8"] = "0"
        Gb, Eb = tb.local_field(Xd)
        del os.environ["HOBO_F8"]
        torch.cuda.synchronize()
        bad = int(((G - Gb).abs().sum(1) > 0).sum())
        st = t.launch_stats()
        print("B", B, "pair", pair, "bad rows", bad, "launches", st["launches"])
