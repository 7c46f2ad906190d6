"""Long randomized parity sweep (diagnostic, not a test): embed (full / region, offsets, views),
binary (wide c, offsets) over random geometries and policies, against the oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1608_00099_b200 as T
from oracle import oracle as O
from triot_inputs import random_shape
DEV = torch.device("cuda:0")

def dev(a, off=0):
    t = torch.from_numpy(np.ascontiguousarray(a))
    buf = torch.empty(t.numel() + off, dtype=t.dtype, device=DEV)
    v = buf[off:].view(t.shape); v.copy_(t.to(DEV)); return v

def bits(a): return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
pols = [(-1, 0), (0, 1), (0, 7), (1, 3), (5, 0)]
bad = 0
for case in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1000):
    dtype = np.float32 if case % 2 else np.float64
    d = int(rng.integers(1, 7))
    shape = random_shape(rng, d, 60000, lo=1, hi=[0, 3000, 250, 40, 15, 8, 6][d])
    if case % 4 == 0:
        shape = shape[:-1] + (int(rng.choice([3, 7, 31, 33, 63, 65, 127, 129, 383, 513, 1000])),)
    T.triot_set_launch_policy(*pols[case % len(pols)])
    src_shape = tuple(max(1, s + int(rng.integers(-3, 3))) for s in shape)
    src = rng.standard_normal(src_shape).astype(dtype)
    region = case % 3 == 1
    ref = np.full(shape, np.nan, dtype=dtype); O.embed(ref, src, region_only=region)
    dst = dev(np.full(shape, np.nan, dtype=dtype), int(rng.integers(0, 4)))
    T.embed(dst, dev(src, int(rng.integers(0, 3))), region_only=region)
    g = dst.cpu().numpy()
    if not np.array_equal(bits(np.nan_to_num(g)), bits(np.nan_to_num(ref))) or \
            not np.array_equal(np.isnan(g), np.isnan(ref)):
        bad += 1; print("EMBED MISMATCH", case, shape, src_shape, region, flush=True)
    # view embed: window of a larger base at a random start
    base = tuple(s + int(rng.integers(0, 5)) for s in shape)
    st = tuple(int(rng.integers(0, b - s + 1)) for b, s in zip(base, shape))
    db = np.full(base, 3.0, dtype=dtype); refv = db.copy()
    sl = tuple(slice(a, a + s) for a, s in zip(st, shape))
    tmp = np.empty(shape, dtype=dtype); O.embed(tmp, src); refv[sl] = tmp
    dbt = dev(db)
    T.embed_view(T.View(dbt, st, shape), T.View(dev(src), None, None))
    if not np.array_equal(bits(dbt.cpu().numpy()), bits(refv)):
        bad += 1; print("VIEW MISMATCH", case, base, st, shape, src_shape, flush=True)
    a = rng.standard_normal(tuple(s + int(rng.integers(0, 2)) for s in shape)).astype(dtype)
    b = rng.standard_normal(tuple(s + int(rng.integers(0, 2)) for s in shape)).astype(dtype)
    cs = tuple(s + int(rng.integers(0, 3)) for s in shape) if case % 2 == 0 else shape
    refc = np.full(cs, 9.0, dtype=dtype); O.apply_binary(a, b, "mul", iter_shape=shape, out=refc)
    c = dev(np.full(cs, 9.0, dtype=dtype), int(rng.integers(0, 3)))
    T.apply_binary(dev(a, int(rng.integers(0, 2))), dev(b), "mul", out=c, iter_shape=shape)
    if not np.array_equal(bits(c.cpu().numpy()), bits(refc)):
        bad += 1; print("BINARY MISMATCH", case, shape, cs, flush=True)
T.triot_set_launch_policy(-1, 0)
print("done, mismatches:", bad)
