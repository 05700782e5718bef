"""PCIe copy rates between device memory and pinned host memory (context for the e2e figures):
one 128 MiB copy per direction, the same split across two streams, and both directions at once."""
import torch

n = 128 << 20
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def split(dst, src):
    cur = torch.cuda.current_stream()
    for i, s in enumerate((s1, s2)):
        s.wait_stream(cur)
        with torch.cuda.stream(s):
            dst[i * n // 2:(i + 1) * n // 2].copy_(src[i * n // 2:(i + 1) * n // 2], non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        h.copy_(d, non_blocking=True)
    with torch.cuda.stream(s2):
        d2.copy_(h2, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


for name, fn, nb in (("d2h", lambda: h.copy_(d, non_blocking=True), n), ("h2d", lambda: d.copy_(h, non_blocking=True), n),
                     ("d2h 2 streams", lambda: split(h, d), n), ("h2d 2 streams", lambda: split(d, h), n),
                     ("d2h + h2d at once", both, 2 * n)):
    ms = timed(fn)
    print(f"{name:18s} {ms:7.3f} ms  {nb / ms / 1e6:6.1f} GB/s")
