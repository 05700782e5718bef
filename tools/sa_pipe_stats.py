"""Pipeline accounting of the persistent annealing kernel on cfg3 (debug build, tools only).
clock64 ticks (about 1.29 per SM cycle on this part; compare ratios, not absolute cycles)."""
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
from workloads import cfg3_problem  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 148 * 128
t = hobo.HoboTensor.from_problem(cfg3_problem())
t0 = t.default_t_start()
t.sa_shard(1, 0, B, 1, t0, t0 / 10)
torch.cuda.synchronize()
L = hobo.lib()
buf = np.zeros((8192, 16), np.uint64)
L.hobo_debug_pipe_stats(buf.ctypes.data_as(C.c_void_p))        # read + clear
t.set_profiling(True)
t.sa_shard(1, 0, B, 1, t0, t0 / 10)
ms = t.launch_stats()["kernel_ms"]
torch.cuda.synchronize()
L.hobo_debug_pipe_stats(buf.ctypes.data_as(C.c_void_p))
n = min(148, (B + 127) // 128)
s = buf[:n].astype(np.float64).mean(axis=0)
sites = 512 * ((B + 127) // 128) / n
tot = s[0]
print(f"kernel {ms:.2f} ms; per CTA: MMA loop {tot:.0f} cyc, {tot / sites:.0f} ticks/site")
print(f"  MMA thread waits: A tiles {s[1] / sites:.0f} ticks/site, W boxes {s[2] / sites:.0f} ticks/site")
print(f"  TMA waiting for free W slots {s[6] / sites:.0f} ticks/site")
print(f"  gen team-0 thread: wait SITE {s[3] / sites:.0f}, decision {s[4] / sites:.0f}, A-gen {s[5] / sites:.0f} "
      f"(of which waiting for free A slots {s[7] / sites:.0f}) ticks/site")
