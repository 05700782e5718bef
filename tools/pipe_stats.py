"""Pipeline accounting of the contraction kernel on cfg3 / cfg3f (debug build, tools only)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2407_19987_b200 import build, hobo  # noqa: E402

dbg = os.path.join(ROOT, "paper_2407_19987_b200", "_lib", "libhobo_dbg.so")
if not os.path.exists(dbg):
    dbg = build.build(debug_stats=True)
hobo.LIB_PATH = dbg
from workloads import cfg3_problem, uniform_colex, x_bits  # noqa: E402

# python tools/pipe_stats.py [cfg3 | cfg3f]   (HOBO_I8 / HOBO_PAIR pick the kernel)
if (sys.argv[1:] or ["cfg3"])[0] == "cfg3f":
    t = hobo.HoboTensor.import_colex(3, 512, uniform_colex(3, 512, 3))
else:
    t = hobo.HoboTensor.from_problem(cfg3_problem())
X = torch.from_numpy(x_bits(3, 65536, 512)).cuda()
G = torch.empty(65536, 512, device="cuda")
E = torch.empty(65536, device="cuda")
t.local_field(X, G, E)
torch.cuda.synchronize()
L = hobo.lib()
buf = np.zeros((8192, 16), np.uint64)
L.hobo_debug_pipe_stats(buf.ctypes.data_as(C.c_void_p))
t.local_field(X, G, E)
torch.cuda.synchronize()
L.hobo_debug_pipe_stats(buf.ctypes.data_as(C.c_void_p))
n = 1024
s = buf[:n].astype(np.float64)
tot = s[:, 0].mean()
kb = s[:, 3].mean()
stg = s[:, 2].mean()
print(f"CTAs {n}: MMA loop {tot:.0f} cyc/CTA, stages {stg:.0f}, K-blocks {kb:.0f}, cyc/kblock {tot/kb:.1f}")
print(f"  MMA thread: wait FULL {s[:,1].mean()/tot*100:5.1f}%  issue {s[:,4].mean()/tot*100:5.1f}%  "
      f"commit {s[:,5].mean()/tot*100:5.1f}%  (per stage: issue {s[:,4].mean()/stg:.0f} cyc, commit {s[:,5].mean()/stg:.0f} cyc)")
print(f"  TMA waiting EMPTY {s[:,6].mean()/tot*100:5.1f}%   generator warp waiting EMPTY {s[:,7].mean()/tot*100:5.1f}%")
print(f"  generator warp 2: A bits {s[:,8].mean()/tot*100:5.1f}%  TMEM store+wait {s[:,9].mean()/tot*100:5.1f}%  "
      f"arrive {s[:,10].mean()/tot*100:5.1f}%  (per stage: bits {s[:,8].mean()/stg:.0f}, store {s[:,9].mean()/stg:.0f}, "
      f"arrive {s[:,10].mean()/stg:.0f}, wait {s[:,7].mean()/stg:.0f} cyc)")
