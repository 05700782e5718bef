"""Probe of the host-buffer paths at one config: device-resident call vs host bytes vs host
packed rows, CUDA-event timed per call (no L2 flush), to see where e2e time goes."""
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2407_19987_b200 import build  # noqa: E402
from paper_2407_19987_b200.hobo import pack_rows  # noqa: E402
from workloads import x_bits  # noqa: E402

build.build()
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
_, factory, N, xseed, B, mode, _ = bench.CONFIGS[cfg]
t = factory()
Xh = torch.from_numpy(x_bits(xseed, B, N)).pin_memory()
Xd = Xh.cuda()
Xp = torch.from_numpy(pack_rows(Xh.numpy()).view(np.int32)).pin_memory()
Xpd = Xp.cuda()
E = torch.empty(B, dtype=torch.float32, device="cuda")
Eh = torch.empty(B, dtype=torch.float32).pin_memory()
s = torch.cuda.current_stream()
field = mode == "field"


def timed(fn, n=10):
    fn()
    torch.cuda.synchronize()
    ms = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        b.synchronize()
        ms.append(a.elapsed_time(b))
    return round(statistics.median(ms), 4), round(min(ms), 4), round(max(ms), 4)


print("device bytes ", timed(lambda: t.energy(Xd, E)))
print("device packed", timed(lambda: t.energy_bits(Xpd, E)))
print("host bytes   ", timed(lambda: t.local_field_host(Xh, Eh, fields=field)))
print("host packed  ", timed(lambda: t.local_field_host_bits(Xp, Eh, fields=field)))
print("h2d packed   ", timed(lambda: Xpd.copy_(Xp, non_blocking=True)))
print("h2d bytes    ", timed(lambda: Xd.copy_(Xh, non_blocking=True)))

# host->device bandwidth by size and buffer: does a small copy run at the PCIe rate?
for mb in (1, 8, 16, 64):
    h = torch.empty(mb << 20, dtype=torch.uint8).pin_memory()
    d = torch.empty(mb << 20, dtype=torch.uint8, device="cuda")
    med = timed(lambda: d.copy_(h, non_blocking=True))[0]
    print(f"h2d {mb:3d} MB fresh pinned: {med} ms = {mb * 1.048576 / med:.1f} GB/s")
h = Xh.view(-1)[: 8 << 20]
d = torch.empty(8 << 20, dtype=torch.uint8, device="cuda")
med = timed(lambda: d.copy_(h, non_blocking=True))[0]
print(f"h2d   8 MB slice of Xh: {med} ms")
