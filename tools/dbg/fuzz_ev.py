"""Randomized expected-value sweep (diagnostic): dense and view windows, every geometry
(vectors, flat, padded view vectors), policies; integer-valued p, so results must be exact."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1608_00099_b200 as T
from oracle import oracle as O
from triot_inputs import random_shape
DEV = torch.device("cuda:0")
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
pols = [(-1, 0), (0, 1), (0, 7), (1, 3), (4, 2), (5, 0)]
bad = 0
for case in range(int(sys.argv[2]) if len(sys.argv) > 2 else 500):
    dtype = np.float32 if case % 2 else np.float64
    d = int(rng.integers(1, 8))
    shape = random_shape(rng, d, 80000, lo=1, hi=[0, 5000, 300, 45, 18, 9, 6, 5][d])
    if case % 3 == 0:
        shape = shape[:-1] + (int(rng.choice([3, 5, 7, 9, 33, 63, 255, 257])),)
    T.triot_set_launch_policy(*pols[case % len(pols)])
    p = rng.integers(0, 64, size=shape).astype(dtype)
    ref = O.expected_value(p)
    off = int(rng.integers(0, 3))
    buf = torch.empty(p.size + off, dtype=torch.from_numpy(p).dtype, device=DEV)
    pt = buf[off:].view(shape); pt.copy_(torch.from_numpy(p).to(DEV))
    m = T.expected_value(pt, with_mass=True).cpu().numpy()
    if not (np.array_equal(m[:-1], ref) and m[-1] == float(p.astype(np.float64).sum())):
        bad += 1; print("EV MISMATCH", case, shape, off, m, ref, flush=True)
    base = tuple(s + int(rng.integers(0, 4)) for s in shape)
    st = tuple(int(rng.integers(0, b - s + 1)) for b, s in zip(base, shape))
    pb = rng.integers(0, 64, size=base).astype(dtype)
    sl = tuple(slice(a, a + s) for a, s in zip(st, shape))
    refv = O.expected_value(np.ascontiguousarray(pb[sl]))
    mv = T.expected_value_view(T.View(torch.from_numpy(pb).to(DEV), st, shape)).cpu().numpy()
    if not np.array_equal(mv, refv):
        bad += 1; print("EV VIEW MISMATCH", case, base, st, shape, mv, refv, flush=True)
T.triot_set_launch_policy(-1, 0)
print("done, mismatches:", bad)
