"""Diagnostic: e4m3-limb fields against the bf16 path, by instance, degree part and batch."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_19987_b200 import hobo as H
from workloads import h, x_bits
from workloads.gen import canonical_cells_all

def pow2_int_cells(order, N, seed, density=0.02):
    idx = canonical_cells_all(order, N)
    cid = h(seed, 1, np.arange(len(idx), dtype=np.uint64), 0)
    keep = (cid % np.uint64(10000)) < np.uint64(int(density * 10000))
    idx = idx[keep]
    r = h(seed, 2, np.arange(len(idx), dtype=np.uint64), 0)
    m = np.array([1, 3, 5, 7], np.int64)[(r % np.uint64(4)).astype(np.int64)]
    e = ((r >> np.uint64(8)) % np.uint64(9)).astype(np.int64)
    sgn = np.where((r >> np.uint64(48)) & np.uint64(1), -1, 1)
    return idx, (sgn * (m << e)).astype(np.float32)

def run(name, make, N, B):
    t = make()
    X = torch.from_numpy(x_bits(17, B, N)).cuda()
    G, E = t.local_field(X)
    kind = t.launch_stats()["i8_planes"]
    os.environ["HOBO_F8"] = "0"
    tb = make()
    Gb, Eb = tb.local_field(X)
    del os.environ["HOBO_F8"]
    torch.cuda.synchronize()
    d = (G != Gb)
    bad = d.nonzero()
    print(name, N, B, "kind", kind, "G bad", int(d.sum()), "E bad", int((E != Eb).sum()),
          "rows", sorted(set(bad[:, 0].tolist()))[:10], "cols", sorted(set(bad[:, 1].tolist()))[:10])

N = 128
idx, val = pow2_int_cells(3, N, 5)
deg = (idx[:, 0] != idx[:, 1]).astype(int) + (idx[:, 1] != idx[:, 2]).astype(int) + 1   # distinct count (sorted idx)
print("cells by degree", np.bincount(deg))
for name, keep in (("all", deg > 0), ("deg3 only", deg == 3), ("deg2 only", deg == 2), ("deg<=2", deg <= 2)):
    ii, vv = idx[keep], val[keep]
    for B in (8, 128):
        run(name, lambda: H.HoboTensor.import_cells(3, N, ii, vv), N, B)

# single candidates: all ones (A = 1 everywhere), and one-hot pairs
ii, vv = idx[deg == 3], val[deg == 3]
t = H.HoboTensor.import_cells(3, N, ii, vv)
os.environ["HOBO_F8"] = "0"
tb = H.HoboTensor.import_cells(3, N, ii, vv)
del os.environ["HOBO_F8"]
pats = {"ones": np.ones(N, bool), "lo": np.arange(N) < 64, "hi": np.arange(N) >= 64, "even": np.arange(N) % 2 == 0,
        "odd": np.arange(N) % 2 == 1, "hi_even": (np.arange(N) >= 64) & (np.arange(N) % 2 == 0),
        "hi_odd": (np.arange(N) >= 64) & (np.arange(N) % 2 == 1), "64-95": (np.arange(N) >= 64) & (np.arange(N) < 96),
        "96-127": np.arange(N) >= 96, "32-95": (np.arange(N) >= 32) & (np.arange(N) < 96),
        "0-31,64-95": (np.arange(N) % 64) < 32, "mod4": np.arange(N) % 4 == 0}
names = list(pats)
X = np.stack([pats[k] for k in names]).astype(np.uint8)
Xd = torch.from_numpy(X).cuda()
G, E = t.local_field(Xd)
os.environ["HOBO_F8"] = "0"
Gb, Eb = tb.local_field(Xd)
del os.environ["HOBO_F8"]
torch.cuda.synchronize()
for r in range(len(names)):
    d = (G[r] - Gb[r]).cpu().numpy()
    print("cand", names[r], "bad cols", int((d != 0).sum()), "first", np.flatnonzero(d)[:10].tolist(), "vals", d[np.flatnonzero(d)[:5]].tolist())

# two-bit candidates: A = 1 for the single tuple {a, b'} (plus the two degree-2 tuples)
prs = [(a, b) for b in range(N) for a in range(b)]
X = np.zeros((len(prs), N), np.uint8)
for r, (a, b) in enumerate(prs):
    X[r, a] = X[r, b] = 1
Xd = torch.from_numpy(X).cuda()
G, E = t.local_field(Xd)
os.environ["HOBO_F8"] = "0"
Gb, Eb = tb.local_field(Xd)
del os.environ["HOBO_F8"]
torch.cuda.synchronize()
bad = ((G - Gb).abs().sum(1) > 0).cpu().numpy()
badp = [prs[i] for i in np.flatnonzero(bad)]
print("two-bit: bad", len(badp), "of", len(prs))
def tindex(a, b):   # colex rank of {a < b} within the degree-3 field segment
    return b * (b - 1) // 2 + a
ks = sorted(tindex(a, b) for a, b in badp)
print("bad tuple K positions", ks[:40], "...", ks[-10:])
print("bad K-blocks (segment)", sorted(set(k // 64 for k in ks)))
print("bad positions within K-block", sorted(set(k % 64 for k in ks))[:64])
