"""GPU parity: the sm_100a kernels (called through the C-ABI) against the CPU oracle.

Bar: bit-exact for embed and apply_binary (memcmp of the whole output),
<= 1e-12 relative per component for the fp64 expected value (against the Neumaier-compensated
oracle), bit-exact for integer-valued and 2^-24-uniform PMFs, and bitwise deterministic.
The five BASELINE configs are compared at full size, element by element, in the same launch
configuration bench.py times (the library chooses it from the shapes and the SM count).
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1608_00099_b200 as T  # noqa: E402
from oracle import oracle as O  # noqa: E402
from triot_inputs import make_inputs, random_shape, random_values, special_values  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def _bits(a: np.ndarray) -> np.ndarray:
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)


def _dev(a: np.ndarray, offset: int = 0):
    """Copy to the GPU; offset > 0 places the tensor `offset` elements into a larger buffer so
    its base pointer is only element-aligned (the alignment fallbacks)."""
    t = torch.from_numpy(np.ascontiguousarray(a))
    if offset == 0:
        return t.to(DEV)
    buf = torch.empty(t.numel() + offset, dtype=t.dtype, device=DEV)
    v = buf[offset:].view(t.shape)
    v.copy_(t.to(DEV))
    return v


def _poisoned(shape, dtype, offset=0):
    x = np.full(shape, np.nan, dtype=dtype)
    return _dev(x, offset)


def assert_bits_equal(got, ref):
    g = got.cpu().numpy()
    assert g.shape == ref.shape
    bad = np.flatnonzero(_bits(g).ravel() != _bits(ref).ravel())
    assert bad.size == 0, f"{bad.size} mismatches, first at flat {bad[:5]}: {g.ravel()[bad[:5]]} vs {ref.ravel()[bad[:5]]}"


# ---------------------------------------------------------------- the five configs, full size

def test_C1_embed_full():
    inp = make_inputs("C1")
    ref = np.empty(inp["dst_shape"]); O.embed(ref, inp["src"])
    dst = _poisoned(inp["dst_shape"], np.float64)
    T.embed(dst, _dev(inp["src"]))
    assert_bits_equal(dst, ref)


def test_C2_embed_full():
    inp = make_inputs("C2")
    ref = np.empty(inp["dst_shape"], np.float32); O.embed(ref, inp["src"])
    dst = _poisoned(inp["dst_shape"], np.float32)
    T.embed(dst, _dev(inp["src"]))
    assert_bits_equal(dst, ref)


def test_C2_embed_misaligned_dst_and_src():
    """C2 with dst (then src) based one element off 32-B alignment: the row-window plan for a
    misaligned output, and the vector plan with element-wise src loads, both bit-exact."""
    inp = make_inputs("C2")
    ref = np.empty(inp["dst_shape"], np.float32); O.embed(ref, inp["src"])
    for off_d, off_s in ((1, 0), (0, 3), (5, 1)):
        dst = _poisoned(inp["dst_shape"], np.float32, off_d)
        T.embed(dst, _dev(inp["src"], off_s))
        assert_bits_equal(dst, ref)


def test_C3_expected_value_full():
    p = make_inputs("C3")["p"]
    ref, plain = O.expected_value(p, with_plain=True)
    pt = _dev(p)
    m1 = T.expected_value(pt).cpu().numpy()
    m2 = T.expected_value(pt).cpu().numpy()
    assert np.all(np.abs(m1 - ref) <= 1e-12 * np.abs(ref)), (m1, ref)
    assert _bits(m1).tolist() == _bits(m2).tolist()          # deterministic run to run


def test_C4_binary_full():
    inp = make_inputs("C4")
    ref = O.apply_binary(inp["a"], inp["b"], "mul", inp["iter_shape"])
    out = T.apply_binary(_dev(inp["a"]), _dev(inp["b"]), "mul")
    assert tuple(out.shape) == inp["iter_shape"]
    assert_bits_equal(out, ref)


def test_C5_embed_full():
    inp = make_inputs("C5")
    ref = np.empty(inp["dst_shape"], np.float32); O.embed(ref, inp["src"])
    dst = _poisoned(inp["dst_shape"], np.float32)
    T.embed(dst, _dev(inp["src"]))
    assert_bits_equal(dst, ref)


def test_region_only_C1_C5():
    for name in ("C1", "C5"):
        inp = make_inputs(name)
        src = inp["src"]
        ref = np.full(inp["dst_shape"], 3.0, dtype=src.dtype)
        O.embed(ref, src, region_only=True)
        dst = _dev(np.full(inp["dst_shape"], 3.0, dtype=src.dtype))
        T.embed(dst, _dev(src), region_only=True)
        assert_bits_equal(dst, ref)


# ---------------------------------------------------------------- random shapes, d = 1..16

def _rand_embed_case(rng, d, dtype):
    hi = 5 if d > 8 else (9 if d > 4 else 40)
    src_shape = random_shape(rng, d, 60000, lo=1, hi=hi)
    dst_shape = tuple(max(0, s + int(rng.integers(-2, 5))) for s in src_shape)
    r = rng.random()
    if r < 0.25:       # tiny / odd innermost extents
        dst_shape = dst_shape[:-1] + (int(rng.choice([1, 2, 3, 4, 5, 8])),)
    elif r < 0.35:     # zero extent somewhere
        k = int(rng.integers(0, d))
        dst_shape = dst_shape[:k] + (0,) + dst_shape[k + 1:]
    if math.prod(dst_shape) > 200000:
        dst_shape = tuple(min(a, b) for a, b in zip(dst_shape, src_shape))
    return src_shape, dst_shape


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("d", list(range(1, 17)))
def test_embed_random(d, dtype):
    rng = np.random.default_rng(10 * d + (dtype == np.float64))
    for rep in range(4):
        src_shape, dst_shape = _rand_embed_case(rng, d, dtype)
        src = rng.standard_normal(src_shape).astype(dtype)
        off_d, off_s = (0, 0) if rep < 2 else (1 + rep % 3, rep % 2)
        for region in (False, True):
            ref = np.full(dst_shape, np.nan, dtype=dtype)
            O.embed(ref, src, region_only=region)
            dst = _poisoned(dst_shape, dtype, off_d)
            T.embed(dst, _dev(src, off_s), region_only=region)
            assert_bits_equal(dst, ref)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("op", ["add", "sub", "mul", "div"])
@pytest.mark.parametrize("d", [1, 2, 3, 4, 5, 6, 8, 11, 14, 16])
def test_binary_random(d, op, dtype):
    rng = np.random.default_rng(100 * d + len(op) + (dtype == np.float64))
    for rep in range(3):
        hi = 5 if d > 8 else (9 if d > 4 else 40)
        ish = random_shape(rng, d, 60000, lo=1, hi=hi)
        if rep == 1:
            ish = ish[:-1] + (int(rng.choice([1, 2, 3, 5])),)
        a = rng.standard_normal(tuple(s + int(rng.integers(0, 3)) for s in ish)).astype(dtype)
        b = rng.standard_normal(tuple(s + int(rng.integers(0, 3)) for s in ish)).astype(dtype)
        cs = tuple(s + int(rng.integers(0, 2)) for s in ish) if rep == 2 else ish
        ref = np.full(cs, 9.0, dtype=dtype)
        O.apply_binary(a, b, op, iter_shape=ish, out=ref)
        out = _dev(np.full(cs, 9.0, dtype=dtype), rep)
        T.apply_binary(_dev(a, rep % 2), _dev(b), op, out=out, iter_shape=ish)
        assert_bits_equal(out, ref)


def test_binary_inplace_and_special_values():
    for dtype in (np.float32, np.float64):
        sv = special_values("f32" if dtype == np.float32 else "f64")
        a = np.tile(sv, 8).reshape(4, 16).astype(dtype)
        b = np.tile(sv[::-1], 8).reshape(4, 16).astype(dtype)
        for op in ("add", "sub", "mul", "div"):
            ref = O.apply_binary(a, b, op)
            at = _dev(a)
            T.apply_binary(at, _dev(b), op, out=at)          # exact in-place c == a
            g = at.cpu().numpy()
            nan = np.isnan(ref)
            assert np.array_equal(np.isnan(g), nan)
            assert_bits_equal(torch.from_numpy(np.where(nan, 0, g)), np.where(nan, 0, ref))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_embed_moves_raw_bits(dtype):
    sv = special_values("f32" if dtype == np.float32 else "f64")
    src = np.tile(sv, 6).reshape(3, 16)
    ref = np.full((5, 19), np.nan, dtype=dtype); O.embed(ref, src)
    dst = _poisoned((5, 19), dtype)
    T.embed(dst, _dev(src))
    assert_bits_equal(dst, ref)


@pytest.mark.parametrize("d", list(range(1, 17)))
def test_ev_random_integer_exact(d):
    rng = np.random.default_rng(500 + d)
    hi = 5 if d > 8 else (9 if d > 4 else 40)
    for rep in range(3):
        shape = random_shape(rng, d, 100000, lo=1, hi=hi)
        if rep == 1:
            shape = shape[:-1] + (int(rng.choice([1, 2, 3, 4])),)
        for dtype in (np.float32, np.float64):
            p = rng.integers(0, 256, size=shape).astype(dtype)
            got = T.expected_value(_dev(p, rep)).cpu().numpy()
            np.testing.assert_array_equal(got, O.expected_value(p))


def test_ev_workspace_reuse_across_grids_and_slots():
    """One workspace (the binding caches one per stream) serves launches of every grid size and
    slot count in turn (other grids, other partial counts, the split-reduction policy): every call
    leaves the arrival counter ready for the next, and partials left by earlier launches are
    never read.  Integer data: every result is exact, so any stale or missing partial shows."""
    rng = np.random.default_rng(91)
    shapes = [(16,) * 5, (3, 4), (64, 64, 64), (2,), (8, 8, 8, 8, 8), (5, 7, 3), (1, 1, 4),
              (128, 96, 48), (4,) * 9, (7, 1, 9), (1000,), (32, 32, 32, 8)]
    cases = []
    for sh in shapes:
        p = rng.integers(0, 64, size=sh).astype(np.float64)
        cases.append((_dev(p), O.expected_value(p), float(p.sum())))
    a = rng.integers(0, 16, size=(40, 30, 20)).astype(np.float64)
    b = rng.integers(0, 16, size=(50, 30, 10)).astype(np.float64)
    ad, bd, dot_ref = _dev(a), _dev(b), float((a[:40, :30, :10] * b[:40, :30, :10]).sum())
    try:
        for rnd in range(6):
            pol = [(-1, 0), (0, 1), (4, 2), (0, 23), (1, 2), (-1, 0)][rnd]
            T.triot_set_launch_policy(*pol)
            for i in rng.permutation(len(cases)):
                pd, ref, mass = cases[i]
                got = T.expected_value(pd, with_mass=True).cpu().numpy()
                np.testing.assert_array_equal(got[:-1], ref)
                assert got[-1] == mass
                if i % 3 == 0:
                    assert float(T.inner_product(ad, bd).cpu()) == dot_ref
    finally:
        T.triot_set_launch_policy(-1, 0)


def test_ev_one_cluster_sizes():
    """Mid-size PMFs (33..256 warp steps) run as one thread-block cluster whose partials meet in
    block 0's shared memory; one block up to 32 steps; the counter path beyond.  Sizes around
    every threshold, both dtypes, with_mass and offsets, the inner product: exact on integer
    data, 1e-12 on real data, identical bits on repeated back-to-back launches."""
    rng = np.random.default_rng(123)
    shapes = [(32, 128), (33, 128), (40, 128), (64, 128), (65, 128), (128, 128), (129, 128),
              (255, 128), (256, 128), (257, 128), (300, 128), (16, 16, 16, 4), (8,) * 5,
              (96, 100), (7, 9, 8, 16)]
    for dtype in (np.float64, np.float32):
        for sh in shapes:
            p = rng.integers(0, 100, size=sh).astype(dtype)
            pd = _dev(p)
            off = tuple(int(x) for x in rng.integers(0, 50, size=len(sh)))
            got = T.expected_value(pd, with_mass=True, offset=off).cpu().numpy()
            ref = O.expected_value(p) + np.array(off, dtype=np.float64) * float(p.sum())
            np.testing.assert_array_equal(got[:-1], ref)
            assert got[-1] == float(p.sum())
            outs = [T.expected_value(pd) for _ in range(6)]   # back to back: PDL + cluster launches
            torch.cuda.synchronize()
            for o in outs:
                np.testing.assert_array_equal(o.cpu().numpy(), O.expected_value(p))
        q = rng.random((100, 128)).astype(dtype)
        g1 = T.expected_value(_dev(q)).cpu().numpy()
        refq = O.expected_value(q)
        assert np.all(np.abs(g1 - refq) <= 1e-12 * np.abs(refq))
        assert _bits(g1).tolist() == _bits(T.expected_value(_dev(q)).cpu().numpy()).tolist()
    a = rng.integers(0, 16, size=(70, 128)).astype(np.float64)
    b = rng.integers(0, 16, size=(64, 160)).astype(np.float64)
    assert float(T.inner_product(_dev(a), _dev(b)).cpu()) == float((a[:64, :128] * b[:64, :128]).sum())


def test_ev_closed_forms():
    p = np.full((16,) * 6, 2.0 ** -24)
    assert T.expected_value(_dev(p)).cpu().tolist() == [7.5] * 6
    q = np.zeros((4, 6, 3, 5)); q[3, 1, 2, 4] = 1.0
    assert T.expected_value(_dev(q)).cpu().tolist() == [3.0, 1.0, 2.0, 4.0]
    e = T.expected_value(_dev(np.zeros((3, 0, 2))))
    assert e.cpu().tolist() == [0.0, 0.0, 0.0]


def test_ev_signed_f32_bound():
    rng = np.random.default_rng(77)
    p = (rng.standard_normal((33, 17, 9, 5))).astype(np.float32)
    ref = O.expected_value(p)
    scale = O.expected_value_abs(p)
    got = T.expected_value(_dev(p)).cpu().numpy()
    assert np.all(np.abs(got - ref) <= 1e-12 * scale)


def test_streams_and_repeated_calls():
    """Several streams, EV workspace ticket left at zero between calls."""
    inp = make_inputs("C1")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    src = _dev(inp["src"])
    ref = np.empty(inp["dst_shape"]); O.embed(ref, inp["src"])
    p = _dev(make_inputs("C3")["p"])
    outs = []
    for s in (s1, s2, s1):
        with torch.cuda.stream(s):
            dst = _poisoned(inp["dst_shape"], np.float64)
            T.embed(dst, src)
            outs.append((dst, T.expected_value(p)))
    torch.cuda.synchronize()
    for dst, m in outs:
        assert_bits_equal(dst, ref)
        assert torch.equal(m, outs[0][1])


def test_prepared_calls():
    """prepare_embed / prepare_apply_binary marshal once; every call of the result issues the same
    C-ABI call on the current stream (bit-exact, also after the inputs change and on a side
    stream); the checks of the plain wrappers run at preparation."""
    inp = make_inputs("C1")
    src = _dev(inp["src"])
    dst = _poisoned(inp["dst_shape"], np.float64)
    call = T.prepare_embed(dst, src)
    ref = np.empty(inp["dst_shape"]); O.embed(ref, inp["src"])
    assert call() is dst
    assert_bits_equal(dst, ref)
    src.mul_(2.0)
    dst.fill_(float("nan"))
    with torch.cuda.stream(torch.cuda.Stream()):
        call()
    torch.cuda.synchronize()
    ref2 = np.empty(inp["dst_shape"]); O.embed(ref2, inp["src"] * 2.0)
    assert_bits_equal(dst, ref2)
    rng = np.random.default_rng(12)
    a, b = rng.standard_normal((9, 14, 6)), rng.standard_normal((12, 10, 8))
    ad, bd = _dev(a), _dev(b)
    bcall = T.prepare_apply_binary(ad, bd, "sub")
    assert_bits_equal(bcall(), O.apply_binary(a, b, "sub"))
    assert_bits_equal(bcall(), O.apply_binary(a, b, "sub"))
    reg = T.prepare_embed(torch.full((6, 6), 7.0, dtype=torch.float64, device=DEV),
                          _dev(np.ones((2, 9))), region_only=True)
    out = reg().cpu().numpy()
    assert out[:2].tolist() == [[1.0] * 6] * 2 and np.all(out[2:] == 7.0)
    with pytest.raises(TypeError):
        T.prepare_embed(dst.cpu(), src.cpu())
    with pytest.raises(ValueError):
        T.prepare_embed(dst, src.float())


def test_errors_raise_not_fallback():
    x = torch.zeros(4, 4, dtype=torch.float64, device=DEV)
    with pytest.raises(T.TriotError):
        T.apply_binary(x, torch.zeros(3, 4, dtype=torch.float64, device=DEV), "mul",
                       iter_shape=(4, 4))
    with pytest.raises(TypeError):
        T.embed(x.cpu(), x.cpu())


@pytest.mark.slow
def test_u64_index_path():
    """A tensor of > 2^32 elements takes the 64-bit-index instances (17.2 GB f32 dst)."""
    free, _ = torch.cuda.mem_get_info()
    if free < 40e9:
        pytest.skip("needs ~20 GB free")
    dst_shape = (65537, 65536)
    src = np.random.default_rng(9).random((5, 70001)).astype(np.float32)
    desc = T.triot_plan_describe(0, [dst_shape, src.shape], None, 2, T.TRIOT_F32, 0)
    assert desc["idx64"]
    dst = torch.full(dst_shape, float("nan"), dtype=torch.float32, device=DEV)
    T.embed(dst, _dev(src))
    torch.cuda.synchronize()
    assert torch.equal(dst[:5, :], torch.from_numpy(src[:, :65536]).to(DEV))
    assert int(torch.count_nonzero(dst[5:])) == 0
    tail = dst[-1, -8:].cpu().numpy()
    assert not np.any(_bits(tail))
    del dst
    torch.cuda.empty_cache()


@pytest.mark.slow
def test_u64_index_path_ev_and_binary():
    """The 64-bit-index instances of the expected value and binary (> 2^32 elements): the EV of
    an all-ones f32 p is exact in fp64, ((n_k - 1) / 2) * N for every axis, and the binary
    product of two formula-generated tensors is checked on sampled elements."""
    free, _ = torch.cuda.mem_get_info()
    if free < 60e9:
        pytest.skip("needs ~55 GB free")
    shape = (65537, 256, 256)          # 4,295,032,832 elements
    n = math.prod(shape)
    desc = T.triot_plan_describe(2, [shape], None, 3, T.TRIOT_F32, 0)
    assert desc["idx64"]
    p = torch.ones(shape, dtype=torch.float32, device=DEV)
    m = T.expected_value(p, with_mass=True).cpu().numpy()
    expect = [(e - 1) / 2 * n for e in shape] + [float(n)]
    np.testing.assert_array_equal(m, np.array(expect))
    del p
    torch.cuda.empty_cache()
    # binary: a[i] = (i mod 1021) / 8, b[i] = (i mod 509) / 16 (exact in f32), c = a * b
    def formula(mod, scale):
        out = torch.empty(n, dtype=torch.float32, device=DEV)
        for s0 in range(0, n, 1 << 29):   # bounded int64 temporaries
            s1 = min(n, s0 + (1 << 29))
            out[s0:s1] = (torch.arange(s0, s1, dtype=torch.int64, device=DEV) % mod).to(
                torch.float32).mul_(scale)
        return out.view(shape)
    a = formula(1021, 0.125)
    b = formula(509, 0.0625)
    c = torch.empty(shape, dtype=torch.float32, device=DEV)
    assert T.triot_plan_describe(1, [shape, shape, shape], None, 3, T.TRIOT_F32, 2)["idx64"]
    T.apply_binary(a, b, "mul", out=c)
    torch.cuda.synchronize()
    idx = np.concatenate([np.arange(64), np.random.default_rng(5).integers(0, n, 4096),
                          np.arange(n - 64, n)])
    got = c.view(-1)[torch.from_numpy(idx).to(DEV)].cpu().numpy()
    ref = ((idx % 1021).astype(np.float32) * np.float32(0.125)) * \
          ((idx % 509).astype(np.float32) * np.float32(0.0625))
    np.testing.assert_array_equal(got, ref)
    del a, b, c
    torch.cuda.empty_cache()


def test_ev_mass_and_slab_amalgamation():
    """triot_expected_value_offset on the slabs of a partition (3 slabs of axis 0, as 3 ranks
    would hold them) summed in slab order by triot_sum_rows equals the oracle on the whole."""
    from paper_1608_00099_b200 import parallel as P
    p = make_inputs("C3")["p"]
    ref = O.expected_value(p)
    full = T.expected_value(_dev(p), with_mass=True).cpu().numpy()
    assert abs(full[6] - math.fsum(p.ravel())) <= 1e-12
    assert np.all(np.abs(full[:6] - ref) <= 1e-12 * np.abs(ref))
    rows = torch.empty((3, 6), dtype=torch.float64, device=DEV)
    for r in range(3):
        lo, hi = P.slab_rows(16, 3, r)
        T.expected_value(_dev(p[lo:hi].copy()), out=rows[r], offset=(lo, 0, 0, 0, 0, 0))
    tot = T.sum_rows(rows).cpu().numpy()
    assert np.all(np.abs(tot - ref) <= 1e-12 * np.abs(ref))
    # integer-valued: exact
    q = np.random.default_rng(3).integers(0, 256, size=(9, 7, 5, 4)).astype(np.float64)
    rows = torch.empty((2, 4), dtype=torch.float64, device=DEV)
    for r in range(2):
        lo, hi = P.slab_rows(9, 2, r)
        T.expected_value(_dev(q[lo:hi].copy()), out=rows[r], offset=(lo, 0, 0, 0))
    np.testing.assert_array_equal(T.sum_rows(rows).cpu().numpy(), O.expected_value(q))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_ev_offset_blocks_of_a_partition(dtype):
    """A random box partition of p (cuts on several axes): each block's EV with its origin as
    offset (weights = global coordinates), summed by triot_sum_rows, equals the oracle on
    the whole p -- exact on integer data, 1e-12 on real data; with_mass puts the block's mass
    last; unit axes (dropped by canonicalisation) still get offset * mass."""
    rng = np.random.default_rng(77 if dtype == np.float32 else 78)
    for trial in range(6):
        d = int(rng.integers(1, 6))
        shape = random_shape(rng, d, 40000, lo=1, hi=12)
        for kind in ("int", "real"):
            p = (rng.integers(0, 64, size=shape).astype(dtype) if kind == "int"
                 else rng.random(shape).astype(dtype))
            ref = O.expected_value(p)
            cuts = [sorted(set([0, int(s)] + [int(c) for c in rng.integers(0, s + 1, size=2)]))
                    for s in shape]
            blocks = [()]
            for k in range(d):
                blocks = [b + ((cuts[k][i], cuts[k][i + 1]),) for b in blocks
                          for i in range(len(cuts[k]) - 1)]
            rows = torch.zeros((len(blocks), d + 1), dtype=torch.float64, device=DEV)
            for i, b in enumerate(blocks):
                sl = tuple(slice(lo, hi) for lo, hi in b)
                blk = np.ascontiguousarray(p[sl])
                if blk.size == 0:
                    continue
                T.expected_value(_dev(blk), out=rows[i], with_mass=True,
                                 offset=tuple(lo for lo, _ in b))
            tot = T.sum_rows(rows).cpu().numpy()
            if kind == "int":
                np.testing.assert_array_equal(tot[:d], ref)
                assert tot[d] == float(p.astype(np.float64).sum())
            else:
                assert np.all(np.abs(tot[:d] - ref) <= 1e-12 * np.abs(ref) + 1e-300), (shape, tot, ref)


def test_sum_rows_order_and_edges():
    rng = np.random.default_rng(5)
    rows = rng.standard_normal((37, 11)) * 10.0 ** rng.integers(-8, 8, size=(37, 11))
    got = T.sum_rows(_dev(rows)).cpu().numpy()
    ref = np.zeros(11)
    for r in range(37):              # rows added in order, fp64 -- bit-exact
        ref = ref + rows[r]
    np.testing.assert_array_equal(got, ref)
    assert T.sum_rows(torch.empty((0, 3), dtype=torch.float64, device=DEV)).cpu().tolist() == [0.0] * 3
    with pytest.raises(T.TriotError):
        x = torch.zeros((4, 4), dtype=torch.float64, device=DEV)
        T._lib.check(T._lib.triot_sum_rows(x.data_ptr(), x.data_ptr(), 4, 4, 0))  # aliasing


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_expected_value_host_streaming(dtype):
    """triot_expected_value_host: p in pinned host memory streamed in chunks through a small
    staging buffer (several chunk axes), per-chunk offset EVs summed in chunk order: equal to the
    oracle (1e-12; exact on integer data), deterministic, with_mass, empty p."""
    p = make_inputs("C3")["p"].astype(dtype)
    ref = O.expected_value(p)
    ph = torch.from_numpy(p).pin_memory()
    for staging_mb in (64, 8, 1):    # 1 MB: chunks of axis 1 rows (prefix over axis 0)
        staging = torch.empty(staging_mb << 20, dtype=torch.uint8, device=DEV)
        got = T.expected_value_host(ph, staging, with_mass=True)
        torch.cuda.synchronize()
        g = got.numpy()
        assert np.all(np.abs(g[:6] - ref) <= 1e-12 * np.abs(ref)), (staging_mb, g, ref)
        assert abs(g[6] - math.fsum(p.astype(np.float64).ravel())) <= 1e-12 * g[6]
        again = T.expected_value_host(ph, staging, with_mass=True)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(again.numpy(), g)
    q = np.random.default_rng(9).integers(0, 256, size=(33, 17, 40, 9)).astype(dtype)
    staging = torch.empty(1 << 20, dtype=torch.uint8, device=DEV)
    got = T.expected_value_host(torch.from_numpy(q).pin_memory(), staging)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(got.numpy(), O.expected_value(q))
    e = T.expected_value_host(torch.from_numpy(np.zeros((3, 0, 4), dtype)), staging, with_mass=True)
    torch.cuda.synchronize()
    assert e.tolist() == [0.0, 0.0, 0.0, 0.0]


# ---------------------------------------------------------------- large real-valued EV parity

@pytest.mark.slow
def test_ev_large_real_f32_2e30():
    """Verdict r1: the telescoped fp64 accumulation at 2^30 real-valued f32 elements, (1024)^3
    uniform[0,1), against the compensated oracle at 1e-12 -- and against the exact value: the
    inputs are multiples of 2^-24, so the marginal sums are exact int64 sums."""
    rng = np.random.default_rng(30)
    q = rng.integers(0, 1 << 24, size=(1024, 1024, 1024), dtype=np.int32)
    p = (q.astype(np.float32) * np.float32(2.0 ** -24))
    got = T.expected_value(_dev(p)).cpu().numpy()
    exact = []
    for k in range(3):
        axes = tuple(j for j in range(3) if j != k)
        marg = q.sum(axis=axes, dtype=np.int64)
        exact.append(int(np.dot(np.arange(1024, dtype=np.int64), marg)))
    ex = np.array([float(e) * 2.0 ** -24 for e in exact])   # ints < 2^63, one rounding each
    assert np.all(np.abs(got - ex) <= 1e-12 * ex), (got, ex)
    ref = O.expected_value(p)
    assert np.all(np.abs(got - ref) <= 1e-12 * np.abs(ref)), (got, ref)
    assert np.all(np.abs(ref - ex) <= 1e-13 * ex)
    del p, q
    torch.cuda.empty_cache()


@pytest.mark.slow
def test_ev_large_signed_f64_and_d16():
    """Signed f64 (512)^3 normal values against the oracle at 1e-12 * sum|t_k p|,
    and a real-valued d = 16 PMF, both deterministic run to run."""
    rng = np.random.default_rng(31)
    p = rng.standard_normal((512, 512, 512))
    got = T.expected_value(_dev(p)).cpu().numpy()
    again = T.expected_value(_dev(p)).cpu().numpy()
    np.testing.assert_array_equal(got, again)
    ref = O.expected_value(p)
    scale = O.expected_value_abs(p)
    assert np.all(np.abs(got - ref) <= 1e-12 * scale), (got, ref)
    q = rng.random((2, 3, 2, 3, 2, 3, 2, 3, 2, 3, 2, 3, 2, 3, 3, 4))
    got = T.expected_value(_dev(q)).cpu().numpy()
    ref = O.expected_value(q)
    assert np.all(np.abs(got - ref) <= 1e-12 * np.abs(ref)), (got, ref)
    del p
    torch.cuda.empty_cache()


@pytest.mark.slow
def test_ev_view_window_of_a_huge_base():
    """an EV view whose window is small but whose span in the base exceeds 2^32
    elements must use 64-bit offsets: base (3, 2^31) f32, window (3, 8) at (0, 5)."""
    n1 = 1 << 31
    base = torch.empty((3, n1), dtype=torch.float32, device=DEV)
    vals = np.arange(24, dtype=np.float32).reshape(3, 8) + 1.0
    base[:, 5:13] = torch.from_numpy(vals).to(DEV)
    got = T.expected_value_view(T.View(base, (0, 5), (3, 8))).cpu().numpy()
    np.testing.assert_array_equal(got, O.expected_value(vals))
    del base
    torch.cuda.empty_cache()


def test_embed_and_binary_slabs_tile_the_result():
    from paper_1608_00099_b200 import parallel as P
    inp = make_inputs("C1")
    ref = np.empty(inp["dst_shape"]); O.embed(ref, inp["src"])
    src = _dev(inp["src"])
    dst = _poisoned(inp["dst_shape"], np.float64)
    for r in range(3):
        lo, hi = P.slab_rows(8, 3, r)
        P.embed_slab(dst[lo:hi], src, lo)
    assert_bits_equal(dst, ref)
    c4 = make_inputs("C4")
    a, b = _dev(c4["a"][:4].copy()), _dev(c4["b"][:4].copy())
    ish = (4,) + c4["iter_shape"][1:]
    refc = O.apply_binary(c4["a"][:4].copy(), c4["b"][:4].copy(), "mul", iter_shape=ish)
    out = torch.empty(ish, dtype=torch.float64, device=DEV)
    for r in range(2):
        lo, hi = P.slab_rows(4, 2, r)
        P.apply_binary_slab(a, b, lo, hi, "mul", out_slab=out[lo:hi], iter_shape=ish)
    assert_bits_equal(out, refc)


def _guarded(shape, dtype, fill, guard=4096, offset=0):
    """A tensor placed between two guard zones of a sentinel bit pattern (writes outside the
    tensor would change them; compute-sanitizer is unavailable on this pool)."""
    n = math.prod(shape)
    buf = torch.full((guard + offset + n + guard,), fill, dtype=dtype, device=DEV)
    return buf, buf[guard + offset: guard + offset + n].view(shape)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_no_writes_outside_outputs(dtype):
    rng = np.random.default_rng(21)
    npdt = np.float32 if dtype == torch.float32 else np.float64
    sentinel = -12345.0
    for case in range(12):
        d = int(rng.integers(1, 15))
        src_shape = random_shape(rng, d, 30000, lo=1, hi=6 if d > 4 else 30)
        dst_shape = tuple(max(1, s + int(rng.integers(-2, 4))) for s in src_shape)
        if case % 3 == 0:
            dst_shape = dst_shape[:-1] + (int(rng.choice([1, 2, 3, 4])),)
        elif case % 3 == 1:   # short odd rows: row windows (element-aligned bases too)
            dst_shape = dst_shape[:-1] + (int(rng.choice([5, 7, 13, 31])),)
        if math.prod(dst_shape) > 100000:
            dst_shape = tuple(min(a, b) for a, b in zip(dst_shape, src_shape))
        src = rng.standard_normal(src_shape).astype(npdt)
        buf, dst = _guarded(dst_shape, dtype, sentinel, offset=case % 3)
        T.embed(dst, _dev(src))
        torch.cuda.synchronize()
        g = 4096 + case % 3
        assert torch.all(buf[:g] == sentinel) and torch.all(buf[g + dst.numel():] == sentinel)
        # binary with c larger than iter: only the iter region of c may change
        ish = tuple(max(1, s - 1) for s in src_shape)
        cs = tuple(s + 1 for s in ish)
        cbuf, c = _guarded(cs, dtype, sentinel, offset=case % 2)
        T.apply_binary(_dev(src), _dev(src), "add", out=c, iter_shape=ish)
        torch.cuda.synchronize()
        g = 4096 + case % 2
        assert torch.all(cbuf[:g] == sentinel) and torch.all(cbuf[g + c.numel():] == sentinel)
        inside = c[tuple(slice(0, s) for s in ish)]
        mask = torch.ones(cs, dtype=torch.bool, device=DEV)
        mask[tuple(slice(0, s) for s in ish)] = False
        assert torch.all(c[mask] == sentinel)
        ref = O.apply_binary(src, src, "add", iter_shape=ish)
        assert_bits_equal(inside.contiguous(), ref)


# ---------------------------------------------------------------- NEXT-1: views

@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("seed", range(10))
def test_views_vs_oracle(seed, dtype):
    rng = np.random.default_rng(7000 + seed)
    d = int(rng.integers(1, 9))
    hi = 7 if d > 4 else 40
    base_a = rng.standard_normal(random_shape(rng, d, 50000, lo=2, hi=hi)).astype(dtype)
    win = tuple(int(rng.integers(1, s + 1)) for s in base_a.shape)
    if seed % 3 == 0:
        win = win[:-1] + (min(base_a.shape[-1], int(rng.choice([1, 2, 3, 4]))),)
    sa = tuple(int(rng.integers(0, s - w + 1)) for s, w in zip(base_a.shape, win))
    base_b = rng.standard_normal(tuple(w + int(rng.integers(0, 3)) for w in win)).astype(dtype)
    sb = tuple(int(rng.integers(0, s - w + 1)) for s, w in zip(base_b.shape, win))
    base_c = np.full(tuple(w + int(rng.integers(0, 3)) for w in win), 7.0, dtype=dtype)
    sc = tuple(int(rng.integers(0, s - w + 1)) for s, w in zip(base_c.shape, win))
    op = ["add", "sub", "mul", "div"][seed % 4]
    ref = base_c.copy()
    O.apply_binary_view(ref, sc, base_a, sa, base_b, sb, win, op)
    c = _dev(base_c)
    T.apply_binary_view(T.View(_dev(base_a), sa, win), T.View(_dev(base_b), sb, win),
                        T.View(c, sc, win), op=op)
    assert_bits_equal(c, ref)
    # embed view -> view (pad/crop), dst base outside its window untouched
    dwin = tuple(max(1, w + int(rng.integers(-1, 3))) for w in win)
    dbase = np.full(tuple(w + 3 for w in dwin), np.nan, dtype=dtype)
    ds = tuple(int(rng.integers(0, 4)) for _ in dwin)
    for region in (False, True):
        refd = dbase.copy()
        O.embed_view(refd, ds, dwin, base_a, sa, win, region_only=region)
        dt = _dev(dbase)
        T.embed_view(T.View(dt, ds, dwin), T.View(_dev(base_a), sa, win), region_only=region)
        assert_bits_equal(dt, refd)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("seed", range(8))
def test_ev_view_vs_oracle(seed, dtype):
    """triot_expected_value_view = Alg 11 on the materialised window (t relative to its start):
    within 1e-12 for real data, exact for integer-valued data, deterministic, mass included."""
    rng = np.random.default_rng(7500 + seed)
    d = int(rng.integers(1, 9))
    hi = 7 if d > 4 else 40
    base = rng.random(random_shape(rng, d, 60000, lo=2, hi=hi)).astype(dtype)
    win = tuple(int(rng.integers(1, s + 1)) for s in base.shape)
    if seed % 3 == 0:   # tiny / odd innermost windows
        win = win[:-1] + (min(base.shape[-1], int(rng.choice([1, 2, 3, 5]))),)
    st = tuple(int(rng.integers(0, s - w + 1)) for s, w in zip(base.shape, win))
    sl = tuple(slice(a, a + w) for a, w in zip(st, win))
    window = np.ascontiguousarray(base[sl])
    ref = O.expected_value(window)
    bdev = _dev(base)
    m1 = T.expected_value_view(T.View(bdev, st, win), with_mass=True).cpu().numpy()
    m2 = T.expected_value_view(T.View(bdev, st, win), with_mass=True).cpu().numpy()
    assert _bits(m1).tolist() == _bits(m2).tolist()
    assert np.all(np.abs(m1[:d] - ref) <= 1e-12 * np.abs(ref) + 1e-300)
    tot = float(window.astype(np.float64).sum())
    assert abs(m1[d] - tot) <= 1e-12 * tot
    # integer-valued: exact
    q = rng.integers(0, 64, size=base.shape).astype(dtype)
    refq = O.expected_value(np.ascontiguousarray(q[sl]))
    np.testing.assert_array_equal(
        T.expected_value_view(T.View(_dev(q), st, win)).cpu().numpy(), refq)


def test_ev_view_whole_base_matches_dense():
    p = make_inputs("C3")["p"]
    dense = T.expected_value(_dev(p)).cpu().numpy()
    view = T.expected_value_view(T.View(_dev(p))).cpu().numpy()
    assert np.all(np.abs(view - dense) <= 1e-12 * np.abs(dense))
    # an interior window of C3's p
    st, win = (2, 0, 3, 1, 0, 4), (12, 16, 9, 15, 16, 7)
    sl = tuple(slice(a, a + w) for a, w in zip(st, win))
    ref = O.expected_value(np.ascontiguousarray(p[sl]))
    got = T.expected_value_view(T.View(_dev(p), st, win)).cpu().numpy()
    assert np.all(np.abs(got - ref) <= 1e-12 * np.abs(ref))


def test_view_centered_fft_padding():
    """The FFT-padding use with the signal placed at an offset: a (384)^3 f32 src embedded
    at (64,64,64) of a (512)^3 dst whose other elements must become +0.0: zero the dst with a
    full embed of an empty window, then embed the src into the interior window."""
    src = make_inputs("C2")["src"]
    dst = torch.full((512,) * 3, float("nan"), dtype=torch.float32, device=DEV)
    T.embed(dst, torch.empty((0, 0, 0), dtype=torch.float32, device=DEV))
    T.embed_view(T.View(dst, (64, 64, 64), (384,) * 3), T.View(_dev(src)))
    torch.cuda.synchronize()
    ref = np.zeros((512,) * 3, np.float32)
    ref[64:448, 64:448, 64:448] = src
    assert_bits_equal(dst, ref)


# ---------------------------------------------------------------- NEXT-2/3: paper Benchmarks 1-3

def test_paper_benchmark1_crop_full():
    from triot_inputs import make_paper_inputs
    inp = make_paper_inputs("B1")
    ref = np.empty(inp["dst_shape"]); O.embed(ref, inp["src"])
    dst = _poisoned(inp["dst_shape"], np.float64)
    T.embed(dst, _dev(inp["src"]))
    assert_bits_equal(dst, ref)


def test_paper_benchmark2_inner_product_full():
    from triot_inputs import make_paper_inputs
    inp = make_paper_inputs("B2")
    ref = O.inner_product(inp["a"], inp["b"])
    a, b = _dev(inp["a"]), _dev(inp["b"])
    g1 = T.inner_product(a, b).item()
    g2 = T.inner_product(a, b).item()
    assert abs(g1 - ref) <= 1e-12 * abs(ref) and g1 == g2


def test_paper_benchmark3_fused_update_full():
    from triot_inputs import make_paper_inputs
    inp = make_paper_inputs("B3")
    ref = inp["x"].copy(); O.fused_update(ref, inp["y"], inp["z"])
    x = _dev(inp["x"])
    T.fused_update(x, _dev(inp["y"]), _dev(inp["z"]))
    assert_bits_equal(x, ref)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("d", [1, 2, 3, 4, 6, 9, 13, 16])
def test_inner_product_and_update_random(d, dtype):
    rng = np.random.default_rng(800 + d + (dtype == np.float64))
    hi = 5 if d > 8 else (9 if d > 4 else 40)
    for rep in range(3):
        ish = random_shape(rng, d, 60000, lo=1, hi=hi)
        if rep == 1:
            ish = ish[:-1] + (int(rng.choice([1, 2, 3, 5])),)
        a = rng.integers(-64, 64, size=tuple(s + int(rng.integers(0, 3)) for s in ish)).astype(dtype)
        b = rng.integers(-64, 64, size=tuple(s + int(rng.integers(0, 3)) for s in ish)).astype(dtype)
        got = T.inner_product(_dev(a, rep % 2), _dev(b), iter_shape=ish).item()
        assert got == O.inner_product(a, b, iter_shape=ish)        # integer-valued: exact
        x = rng.standard_normal(ish).astype(dtype)
        y = rng.standard_normal(tuple(s + int(rng.integers(0, 3)) for s in ish)).astype(dtype)
        z = rng.standard_normal(tuple(s + int(rng.integers(0, 3)) for s in ish)).astype(dtype)
        ref = x.copy(); O.fused_update(ref, y, z)
        xt = _dev(x, rep)
        T.fused_update(xt, _dev(y), _dev(z))
        assert_bits_equal(xt, ref)
    # empty iteration -> 0.0
    e = T.inner_product(_dev(np.zeros((0,) * d, dtype)), _dev(np.zeros((2,) * d, dtype)))
    assert e.item() == 0.0


# ---------------------------------------------------------------- NEXT-4: naive convolution

def test_paper_benchmark4_convolution():
    """Benchmark 4: two (2^8, 2^3) matrices; bit-identical to Alg 15."""
    rng = np.random.default_rng(17)
    lhs, rhs = rng.random((256, 8)), rng.random((256, 8))
    ref = O.naive_convolve(lhs, rhs)
    got = T.naive_convolve(_dev(lhs), _dev(rhs))
    assert tuple(got.shape) == (511, 15)
    assert_bits_equal(got, ref)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("d", [1, 2, 3, 4, 5, 7, 10])
def test_convolution_random(d, dtype):
    rng = np.random.default_rng(900 + d + (dtype == np.float32))
    for rep in range(2):
        ls = random_shape(rng, d, 3000 if d < 5 else 600, lo=1, hi=6 if d > 3 else 14)
        rs = random_shape(rng, d, 600 if d < 5 else 200, lo=1, hi=5 if d > 3 else 10)
        lhs = rng.standard_normal(ls).astype(dtype)
        rhs = rng.standard_normal(rs).astype(dtype)
        # larger lhs: the lane kernel iterates rhs in reverse; swapped: lhs forward
        for x, y in ((lhs, rhs), (rhs, lhs)):
            ref = O.naive_convolve(x, y)
            try:
                for mode in (-1, 0, 1):   # automatic / lane per output / G-lane groups
                    T.triot_set_launch_policy(mode, 0)
                    got = T.naive_convolve(_dev(x, rep), _dev(y))
                    assert_bits_equal(got, ref)
            finally:
                T.triot_set_launch_policy(-1, 0)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_convolution_global_operands(dtype):
    """Operands too large for shared-memory staging (> 96 KB together): global loads."""
    rng = np.random.default_rng(77)
    m = 2 if dtype == np.float32 else 1
    for ls, rs in (((300 * m, 41), (7, 9)), ((5, 6), (200 * m, 70))):
        lhs = rng.standard_normal(ls).astype(dtype)
        rhs = rng.standard_normal(rs).astype(dtype)
        ref = O.naive_convolve(lhs, rhs)
        try:
            for mode in (-1, 0, 1):
                T.triot_set_launch_policy(mode, 0)
                assert_bits_equal(T.naive_convolve(_dev(lhs), _dev(rhs)), ref)
        finally:
            T.triot_set_launch_policy(-1, 0)


# ---------------------------------------------------------------- host-buffer streaming

def test_host_streaming_embed_and_binary():
    from paper_1608_00099_b200 import api
    for name in ("C1", "C2", "C5"):      # C5: one axis-0 row of dst is 268 MB -> chunks of axis k>0
        inp = make_inputs(name)
        ref = np.empty(inp["dst_shape"], inp["src"].dtype); O.embed(ref, inp["src"])
        src = torch.from_numpy(inp["src"]).pin_memory()
        dst = torch.full(inp["dst_shape"], float("nan"), dtype=src.dtype).pin_memory()
        T.embed_host(dst, src)
        torch.cuda.synchronize()
        assert_bits_equal(dst, ref)
    # small staging forces many slabs and slot reuse
    inp = make_inputs("C4")
    a, b = torch.from_numpy(inp["a"][:9].copy()).pin_memory(), torch.from_numpy(inp["b"][:9].copy()).pin_memory()
    ish = (9,) + inp["iter_shape"][1:]
    ref = O.apply_binary(inp["a"][:9].copy(), inp["b"][:9].copy(), "mul", iter_shape=ish)
    old = api.STAGING_BYTES
    try:
        api._ws_cache.clear()
        api.STAGING_BYTES = 64 << 20        # two slots of 32 MB: ~1 row of a + b + c per slab
        out = T.apply_binary_host(a, b, "mul", iter_shape=ish)
        torch.cuda.synchronize()
    finally:
        api.STAGING_BYTES = old
        api._ws_cache.clear()
    assert_bits_equal(out, ref)


@pytest.mark.parametrize("dst_shape,src_shape,dtype", [
    ((4,) * 9, (3,) * 9, np.float32),
    ((5, 4, 4, 2, 8), (2, 3, 4, 2, 5), np.float32),
    ((3, 6, 2, 4, 4, 4), (3, 4, 1, 3, 2, 4), np.float64),
    ((7, 3, 4, 4, 4, 4), (7, 3, 4, 4, 3, 3), np.float32),  # zero runs of one step only
])
def test_embed_zero_runs(dst_shape, src_shape, dtype):
    """Shapes whose plan stores zero runs without the odometer, under several chunkings (runs
    cut by chunk ends, ragged last step), bit-exact against the oracle."""
    rng = np.random.default_rng(91)
    src = rng.standard_normal(src_shape).astype(dtype)
    ref = np.empty(dst_shape, dtype); O.embed(ref, src)
    try:
        for mode, bpsm in [(-1, 0), (0, 1), (0, 3), (0, 200)]:
            T.triot_set_launch_policy(mode, bpsm)
            dst = _poisoned(dst_shape, dtype)
            T.embed(dst, _dev(src))
            assert_bits_equal(dst, ref)
    finally:
        T.triot_set_launch_policy(-1, 0)


def test_results_independent_of_launch_policy():
    """Every work decomposition gives bit-identical embed / binary / dot / update results, and the
    expected value stays deterministic per policy and within 1e-12 across policies."""
    rng = np.random.default_rng(55)
    src = rng.standard_normal((37, 29, 11)).astype(np.float32)
    a = rng.standard_normal((33, 17, 9, 6)); b = rng.standard_normal((35, 17, 12, 8))
    ps = [rng.random((13, 7, 9, 5)), rng.random((9, 16, 8, 12))]  # flat / 32-B vectors
    ref_e = np.empty((41, 32, 12), np.float32); O.embed(ref_e, src)
    ref_b = O.apply_binary(a, b, "div")
    ref_ms = [O.expected_value(p) for p in ps]
    try:
        for mode, bpsm in [(0, 1), (0, 7), (0, 64), (1, 1), (1, 3), (2, 1), (3, 2), (4, 1),
                           (4, 16), (4, 64), (-1, 0)]:
            T.triot_set_launch_policy(mode, bpsm)
            dst = _poisoned((41, 32, 12), np.float32)
            T.embed(dst, _dev(src))
            assert_bits_equal(dst, ref_e)
            assert_bits_equal(T.apply_binary(_dev(a), _dev(b), "div"), ref_b)
            for p, ref_m in zip(ps, ref_ms):
                m1 = T.expected_value(_dev(p), with_mass=True).cpu().numpy()
                m2 = T.expected_value(_dev(p), with_mass=True).cpu().numpy()
                assert _bits(m1).tolist() == _bits(m2).tolist()
                assert np.all(np.abs(m1[:-1] - ref_m) <= 1e-12 * np.abs(ref_m))
                assert abs(m1[-1] - p.sum()) <= 1e-12 * p.sum()
    finally:
        T.triot_set_launch_policy(-1, 0)


# ---------------------------------------------------------------- row windows (short odd rows)

@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("seed", range(8))
def test_row_windows_vs_oracle(seed, dtype):
    """Short odd innermost extents (row-window kernels) for embed (pad, crop, region only) and
    every binary op (dense and strided c, element-aligned bases), bit-exact; the same calls with
    row windows switched off (flat vectors, policy mode 5) give the same bits."""
    rng = np.random.default_rng(700 + seed)
    d = int(rng.integers(1, 8))
    n = int(rng.choice([1, 3, 5, 7, 9, 13, 31, 33, 63]))
    outer = random_shape(rng, d - 1, 40000 // max(n, 4), lo=1, hi=40 if d <= 3 else 7) if d > 1 else ()
    dst_shape = outer + (n,)
    src_shape = tuple(max(1, s + int(rng.integers(-2, 3))) for s in dst_shape)
    src = rng.standard_normal(src_shape).astype(dtype)
    a = rng.standard_normal(tuple(s + int(rng.integers(0, 3)) for s in dst_shape)).astype(dtype)
    b = rng.standard_normal(tuple(s + int(rng.integers(0, 3)) for s in dst_shape)).astype(dtype)
    op = ["add", "sub", "mul", "div"][seed % 4]
    try:
        for mode in (-1, 5):
            T.triot_set_launch_policy(mode, 0)
            for region, off in ((False, 0), (True, 1), (False, 3)):
                ref = np.full(dst_shape, np.nan, dtype=dtype)
                O.embed(ref, src, region_only=region)
                dst = _poisoned(dst_shape, dtype, off)
                T.embed(dst, _dev(src, off % 2), region_only=region)
                assert_bits_equal(dst, ref)
            for cs, off in ((dst_shape, 0), (tuple(s + 1 for s in dst_shape), 1)):
                ref = np.full(cs, 9.0, dtype=dtype)
                O.apply_binary(a, b, op, iter_shape=dst_shape, out=ref)
                out = _dev(np.full(cs, 9.0, dtype=dtype), off)
                T.apply_binary(_dev(a, off), _dev(b), op, out=out, iter_shape=dst_shape)
                assert_bits_equal(out, ref)
            x = rng.standard_normal(dst_shape).astype(dtype)
            ref = O.apply_binary(x, b, op, iter_shape=dst_shape)
            xt = _dev(x)
            T.apply_binary(xt, _dev(b), op, out=xt, iter_shape=dst_shape)   # in place, c == a
            assert_bits_equal(xt, ref)
    finally:
        T.triot_set_launch_policy(-1, 0)


def test_row_windows_large_and_policies():
    """A large short-odd-row embed / binary (many windows per warp, all-zero windows, ragged last
    window) under every decomposition, bit-exact against the oracle."""
    rng = np.random.default_rng(71)
    src = rng.standard_normal((700, 300, 5)).astype(np.float32)
    ref = np.empty((733, 310, 7), np.float32); O.embed(ref, src)
    a = rng.standard_normal((701, 311, 7)); b = rng.standard_normal((700, 310, 9))
    refb = O.apply_binary(a, b, "mul", iter_shape=(700, 310, 7))
    try:
        for mode, bpsm in [(-1, 0), (0, 1), (0, 5), (1, 1), (1, 7), (0, 300)]:
            T.triot_set_launch_policy(mode, bpsm)
            dst = _poisoned((733, 310, 7), np.float32)
            T.embed(dst, _dev(src))
            assert_bits_equal(dst, ref)
            out = T.apply_binary(_dev(a), _dev(b), "mul", iter_shape=(700, 310, 7))
            assert_bits_equal(out, refb)
    finally:
        T.triot_set_launch_policy(-1, 0)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_row_windows_long_odd_rows_non_dense_outputs(dtype):
    """Odd rows past the dense thresholds into non-dense outputs (a view window at an odd
    offset, region-only embed, c wider than the iteration), bit-exact against the oracle."""
    rng = np.random.default_rng(97)
    src = rng.standard_normal((41, 19, 383)).astype(dtype)
    # view: src window (37,17,381) at (1,1,1) into dst base (45,23,401) at (3,5,7)
    dbase = np.full((45, 23, 401), 3.0, dtype=dtype)
    ref = dbase.copy()
    ref[3:40, 5:22, 7:388] = src[1:38, 1:18, 1:382]
    db = _dev(dbase)
    T.embed_view(T.View(db, (3, 5, 7), (37, 17, 381)), T.View(_dev(src), (1, 1, 1), (37, 17, 381)))
    assert_bits_equal(db, ref)
    # region only, dst rows of 401 over src rows of 383 (pre-filled dst keeps its padding)
    dst = _dev(np.full((45, 23, 401), 3.0, dtype=dtype), 1)
    ref = np.full((45, 23, 401), 3.0, dtype=dtype)
    O.embed(ref, src, region_only=True)
    T.embed(dst, _dev(src), region_only=True)
    assert_bits_equal(dst, ref)
    # binary, c wider than the iteration: rows of 99 (row table) and of 199 (a warp per row)
    for n in (99, 199):
        a = rng.standard_normal((40, 17, n)).astype(dtype)
        b = rng.standard_normal((41, 18, n)).astype(dtype)
        ref = np.full((40, 17, 300), 9.0, dtype=dtype)
        O.apply_binary(a, b, "sub", iter_shape=(40, 17, n), out=ref)
        c = _dev(np.full((40, 17, 300), 9.0, dtype=dtype), 1)
        T.apply_binary(_dev(a), _dev(b), "sub", out=c, iter_shape=(40, 17, n))
        assert_bits_equal(c, ref)


@pytest.mark.slow
def test_u64_index_path_row_windows():
    """The 64-bit-index row-window instance: embed f32 (613566757, 7) <- (613566757, 5), 4.3 G
    destination elements, src generated by a formula, checked on the device in slabs."""
    free, _ = torch.cuda.mem_get_info()
    if free < 45e9:
        pytest.skip("needs ~32 GB free")
    rows = 613566757
    desc = T.triot_plan_describe(0, [(rows, 7), (rows, 5)], None, 2, T.TRIOT_F32, 0)
    assert desc["idx64"] and desc["rows"]
    src = torch.empty((rows, 5), dtype=torch.float32, device=DEV)
    flat = src.view(-1)
    for s0 in range(0, flat.numel(), 1 << 29):
        s1 = min(flat.numel(), s0 + (1 << 29))
        flat[s0:s1] = (torch.arange(s0, s1, dtype=torch.int64, device=DEV) % 1021).to(
            torch.float32) / 8
    dst = torch.full((rows, 7), float("nan"), dtype=torch.float32, device=DEV)
    T.embed(dst, src)
    torch.cuda.synchronize()
    for r0 in range(0, rows, 1 << 26):
        r1 = min(rows, r0 + (1 << 26))
        assert torch.equal(dst[r0:r1, :5], src[r0:r1])
        assert int(torch.count_nonzero(dst[r0:r1, 5:])) == 0
    del dst, src, flat
    torch.cuda.empty_cache()


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("seed", range(6))
def test_ev_odd_innermost_vs_oracle(seed, dtype):
    """Expected value over short odd innermost extents (flat vectors, closed-form in-vector
    weights): integer-valued p exact, real p within 1e-12, mass included, deterministic, and the
    same under policy mode 5."""
    rng = np.random.default_rng(900 + seed)
    d = int(rng.integers(1, 7))
    n = int(rng.choice([3, 5, 7, 9, 11, 13, 15]))
    outer = random_shape(rng, d - 1, 200000 // n, lo=1, hi=30 if d <= 3 else 9) if d > 1 else ()
    shape = outer + (n,)
    pi = rng.integers(0, 256, size=shape).astype(dtype)
    m = T.expected_value(_dev(pi), with_mass=True).cpu().numpy()
    np.testing.assert_array_equal(m[:-1], O.expected_value(pi))
    assert m[-1] == float(pi.astype(np.float64).sum())
    pr = rng.random(shape).astype(dtype)
    ref = O.expected_value(pr)
    m1 = T.expected_value(_dev(pr)).cpu().numpy()
    m2 = T.expected_value(_dev(pr)).cpu().numpy()
    assert _bits(m1).tolist() == _bits(m2).tolist()
    assert np.all(np.abs(m1 - ref) <= 1e-12 * np.abs(ref))
    try:
        T.triot_set_launch_policy(5, 0)
        mf = T.expected_value(_dev(pr)).cpu().numpy()
    finally:
        T.triot_set_launch_policy(-1, 0)
    assert np.all(np.abs(mf - ref) <= 1e-12 * np.abs(ref))


def test_fuzz_embed_binary_geometries():
    """A randomized sweep over every geometry the planner can pick (32-B / 16-B / element
    vectors, collapsed rows, flat vectors, row windows, zero runs, 64 dims of odd and even
    extents), with element-aligned bases, region-only embeds, wide outputs and random launch
    policies: every output bit-exact against the oracle."""
    rng = np.random.default_rng(2024)
    policies = [(-1, 0), (0, 1), (0, 3), (1, 2), (5, 0)]
    try:
        for case in range(240):
            dtype = np.float32 if case % 2 else np.float64
            d = int(rng.integers(1, 9)) if case % 8 else int(rng.integers(9, 17))
            shape = random_shape(rng, d, 20000, lo=1, hi=40 if d <= 2 else (12 if d <= 4 else
                                                                           (5 if d <= 8 else 3)))
            if case % 5 == 0:
                shape = shape[:-1] + (int(rng.choice([3, 5, 7, 9, 31, 33, 65])),)
            src_shape = tuple(max(1, s + int(rng.integers(-2, 3))) for s in shape)
            T.triot_set_launch_policy(*policies[case % len(policies)])
            region = case % 3 == 1
            off_d, off_s = int(rng.integers(0, 3)), int(rng.integers(0, 2))
            src = rng.standard_normal(src_shape).astype(dtype)
            ref = np.full(shape, np.nan, dtype=dtype)
            O.embed(ref, src, region_only=region)
            dst = _poisoned(shape, dtype, off_d)
            T.embed(dst, _dev(src, off_s), region_only=region)
            got = dst.cpu().numpy()
            if region:   # untouched elements stay NaN-poisoned on both sides
                assert np.array_equal(np.isnan(got), np.isnan(ref))
                got, ref = np.nan_to_num(got), np.nan_to_num(ref)
            assert np.array_equal(_bits(got), _bits(ref)), (case, shape, src_shape, region)
            a = rng.standard_normal(tuple(s + int(rng.integers(0, 2)) for s in shape)).astype(dtype)
            b = rng.standard_normal(tuple(s + int(rng.integers(0, 2)) for s in shape)).astype(dtype)
            cs = tuple(s + int(rng.integers(0, 2)) for s in shape) if case % 4 == 0 else shape
            op = ["add", "sub", "mul", "div"][case % 4]
            refc = np.full(cs, 9.0, dtype=dtype)
            O.apply_binary(a, b, op, iter_shape=shape, out=refc)
            c = _dev(np.full(cs, 9.0, dtype=dtype), int(rng.integers(0, 2)))
            T.apply_binary(_dev(a, int(rng.integers(0, 2))), _dev(b), op, out=c, iter_shape=shape)
            assert_bits_equal(c, refc)
    finally:
        T.triot_set_launch_policy(-1, 0)


def test_sharded_expected_value_over_nccl():
    """The slab-sharded expected value (paper_1608_00099_b200/parallel.py) with the real kernel
    and the NCCL backend (world size 1 on this one-GPU box: the collective path runs for real),
    equal to the single-call result within 1e-12 and exact on integer data."""
    import os
    import socket
    import torch.distributed as dist
    from paper_1608_00099_b200 import parallel as P
    if dist.is_initialized():
        pytest.skip("a process group already exists")
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=DEV)
    try:
        p = make_inputs("C3")["p"]
        pi = np.random.default_rng(3).integers(0, 256, size=(9, 7, 16, 8)).astype(np.float64)
        for arr, exact in ((pi, True), (p, False)):
            ref = O.expected_value(arr)
            lo, hi = P.slab_rows(arr.shape[0], 1, 0)
            got = P.expected_value_sharded(_dev(arr[lo:hi].copy()), lo).cpu().numpy()
            if exact:
                np.testing.assert_array_equal(got, ref)
            else:
                assert np.all(np.abs(got - ref) <= 1e-12 * np.abs(ref))
    finally:
        dist.destroy_process_group()


def test_misaligned_merged_outputs():
    """A fully merged pad into a dst one element off the 32-byte grid and a merged binary into a
    misaligned c (both shifted 32-B stores), bit-exact against the oracle."""
    rng = np.random.default_rng(33)
    src = rng.standard_normal((500, 512, 512)).astype(np.float32)
    desc = T.triot_plan_describe(0, [(512, 512, 512), src.shape], None, 3, T.TRIOT_F32, 0,
                                 (4, 0, 0))
    assert desc["dshift"] == 1
    ref = np.empty((512, 512, 512), np.float32)
    O.embed(ref, src)
    dst = _poisoned((512, 512, 512), np.float32, 1)
    T.embed(dst, _dev(src))
    assert_bits_equal(dst, ref)
    del dst
    a = rng.standard_normal((256, 512, 512)).astype(np.float32)
    b = rng.standard_normal((256, 512, 512)).astype(np.float32)
    desc = T.triot_plan_describe(1, [a.shape, a.shape, b.shape], None, 3, T.TRIOT_F32, 2,
                                 (4, 0, 0))
    assert desc["dshift"] == 1
    refc = O.apply_binary(a, b, "mul")
    c = _dev(np.zeros(a.shape, np.float32), 1)
    T.apply_binary(_dev(a), _dev(b), "mul", out=c)
    assert_bits_equal(c, refc)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_ev_view_odd_windows(dtype):
    """Expected value of view windows whose rows take no vector width (odd lengths >= 32, odd
    starts): integer-valued data exact, real data within 1e-12, the mass, deterministic."""
    rng = np.random.default_rng(61)
    for base, start, win in [((40, 70, 300), (3, 5, 7), (33, 61, 255)),
                             ((9, 300), (1, 1), (8, 297)),
                             ((4, 5, 6, 200), (1, 0, 2, 3), (3, 5, 4, 33)),
                             ((2000,), (3,), (1901,))]:
        for kind in ("int", "real"):
            if kind == "int":
                b = rng.integers(0, 256, size=base).astype(dtype)
            else:
                b = rng.random(base).astype(dtype)
            sl = tuple(slice(s, s + w) for s, w in zip(start, win))
            ref = O.expected_value(np.ascontiguousarray(b[sl]))
            bt = _dev(b)
            m1 = T.expected_value_view(T.View(bt, start, win), with_mass=True).cpu().numpy()
            m2 = T.expected_value_view(T.View(bt, start, win), with_mass=True).cpu().numpy()
            assert _bits(m1).tolist() == _bits(m2).tolist()
            if kind == "int":
                np.testing.assert_array_equal(m1[:-1], ref)
                assert m1[-1] == float(b[sl].astype(np.float64).sum())
            else:
                assert np.all(np.abs(m1[:-1] - ref) <= 1e-12 * np.abs(ref)), (m1, ref)



@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_shifted_stores_every_offset(dtype):
    """Embeds into a dense dst at every element offset from the 32-byte grid (shifted 32-B
    stores: partial head / tail chunks per warp step, ragged last steps, collapsed rows, zero
    vectors), bit-exact against the oracle under several decompositions."""
    rng = np.random.default_rng(44)
    V = 32 // np.dtype(dtype).itemsize
    cases = [((37, 29, 16), (33, 30, 11)), ((9, 64), (8, 70)), ((5, 6, 4, 4), (4, 5, 3, 4)),
             ((3, 1000), (3, 999))]
    try:
        for mode, bpsm in [(-1, 0), (0, 1), (1, 2)]:
            T.triot_set_launch_policy(mode, bpsm)
            for dst_shape, src_shape in cases:
                src = rng.standard_normal(src_shape).astype(dtype)
                ref = np.empty(dst_shape, dtype); O.embed(ref, src)
                for off in range(1, V):
                    dst = _poisoned(dst_shape, dtype, off)
                    T.embed(dst, _dev(src, off % 2))
                    assert_bits_equal(dst, ref)
    finally:
        T.triot_set_launch_policy(-1, 0)



@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_binary_shifted_stores_every_offset(dtype):
    """Binary ops into a dense c at every element offset from the 32-byte grid (shifted 32-B
    stores), including exact in place (c == a), bit-exact against the oracle."""
    rng = np.random.default_rng(45)
    V = 32 // np.dtype(dtype).itemsize
    for ish, ash, bsh in [((37, 29, 16), (37, 30, 16), (38, 29, 24)), ((9, 64), (9, 64), (9, 64)),
                          ((3, 1000), (3, 1000), (4, 1000))]:
        a = rng.standard_normal(ash).astype(dtype)
        b = rng.standard_normal(bsh).astype(dtype)
        for op in ("add", "div"):
            ref = O.apply_binary(a, b, op, iter_shape=ish)
            for off in range(1, V):
                c = _dev(np.full(ish, 9.0, dtype=dtype), off)
                T.apply_binary(_dev(a), _dev(b), op, out=c, iter_shape=ish)
                assert_bits_equal(c, ref)
                if ash == ish:   # in place: a misaligned by the same offset, c == a
                    at = _dev(a, off)
                    T.apply_binary(at, _dev(b), op, out=at, iter_shape=ish)
                    assert_bits_equal(at, ref)


@pytest.mark.slow
def test_u64_index_path_shifted_stores():
    """The 64-bit-index shifted-store instance: a 4.3 G-element f32 dst one element off the
    32-byte grid, checked on the device."""
    free, _ = torch.cuda.mem_get_info()
    if free < 40e9:
        pytest.skip("needs ~20 GB free")
    dst_shape = (65537, 65536)
    src = np.random.default_rng(19).random((5, 70001)).astype(np.float32)
    desc = T.triot_plan_describe(0, [dst_shape, src.shape], None, 2, T.TRIOT_F32, 0, (4, 0, 0))
    assert desc["idx64"] and desc["dshift"] == 1
    buf = torch.full((65537 * 65536 + 1,), float("nan"), dtype=torch.float32, device=DEV)
    dst = buf[1:].view(dst_shape)
    T.embed(dst, _dev(src))
    torch.cuda.synchronize()
    assert torch.isnan(buf[0])                      # the element before dst is untouched
    assert torch.equal(dst[:5, :], torch.from_numpy(src[:, :65536]).to(DEV))
    for r0 in range(5, 65537, 8192):
        assert int(torch.count_nonzero(dst[r0:r0 + 8192])) == 0
    del dst, buf
    torch.cuda.empty_cache()


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_view_embed_long_rows_vectorized(dtype):
    """Embeds into view windows at odd offsets whose rows are long and a multiple of the vector
    width (a warp per row moving 32-B vectors, stores shifted to the 32-byte grid; partial last
    vector groups), including src windows narrower than dst (zero padding), bit-exact."""
    rng = np.random.default_rng(64)
    for dbase, dstart, win, sw in [((24, 36, 300), (1, 3, 5), (20, 30, 256), 256),
                                   ((9, 1100), (2, 7), (6, 1024), 1000),
                                   ((5, 7, 520), (0, 1, 3), (4, 5, 512), 512)]:
        src = rng.standard_normal(win[:-1] + (sw,)).astype(dtype)
        db = np.full(dbase, 3.0, dtype=dtype)
        ref = db.copy()
        sl = tuple(slice(a, a + w) for a, w in zip(dstart, win))
        tmp = np.empty(win, dtype=dtype)
        O.embed(tmp, src)
        ref[sl] = tmp
        dbt = _dev(db)
        T.embed_view(T.View(dbt, dstart, win), T.View(_dev(src)))
        assert_bits_equal(dbt, ref)


def test_plan_cache_pointers_alignment_and_aliasing():
    """The host plan cache (dense embed / binary) keys on shapes, dtype, op, alignment and
    policy: repeated calls with new buffers stay bit-exact, a call whose buffers overlap after a
    cached disjoint call is still refused (or run in place when allowed), and a misaligned call
    after an aligned one takes its own plan."""
    inp = make_inputs("C1")
    ref = np.empty(inp["dst_shape"]); O.embed(ref, inp["src"])
    src = _dev(inp["src"])
    for _ in range(3):                       # fresh dst buffers, same key: cached plan
        dst = _poisoned(inp["dst_shape"], np.float64)
        T.embed(dst, src)
        assert_bits_equal(dst, ref)
    for off in (1, 2, 0):                    # alignment changes the key
        dst = _poisoned(inp["dst_shape"], np.float64, off)
        T.embed(dst, _dev(inp["src"], (off + 1) % 3))
        assert_bits_equal(dst, ref)
    # overlap after a cached disjoint call: dst over src's buffer is refused
    buf = torch.zeros(2 * 8 * 16 * 8 * 8 + 4 * 9 * 7 * 5, dtype=torch.float64, device=DEV)
    d1 = buf[:8192].view(8, 16, 8, 8)
    s1 = buf[8192:8192 + 1260].view(4, 9, 7, 5)
    s1.copy_(src)
    T.embed(d1, s1)                           # disjoint: cached
    assert_bits_equal(d1, ref)
    s2 = buf[100:100 + 1260].view(4, 9, 7, 5)     # elements [100, 1360)
    with pytest.raises(T.TriotError, match="ALIASING"):   # dst [1000, 9192) overlaps it
        T.embed(buf[1000:1000 + 8192].view(8, 16, 8, 8), s2)
    # binary: out-of-place (cached), then exact in place on the same shapes (allowed)
    rng = np.random.default_rng(4)
    a = rng.random((7, 9, 16)); b = rng.random((7, 9, 16))
    refc = O.apply_binary(a, b, "mul")
    ta, tb = _dev(a), _dev(b)
    for _ in range(2):
        c = T.apply_binary(ta, tb, "mul")
        assert_bits_equal(c, refc)
    T.apply_binary(ta, tb, "mul", out=ta)     # c == a: in place
    assert_bits_equal(ta, refc)
    with pytest.raises(T.TriotError, match="ALIASING"):   # partial overlap: refused
        big = torch.zeros(2 * 7 * 9 * 16, dtype=torch.float64, device=DEV)
        T.apply_binary(big[:1008].view(7, 9, 16), tb, "mul", out=big[8:1016].view(7, 9, 16))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_ev_row_tiles_vs_oracle(dtype):
    """The dense EV of short odd rows (ev_rows_kernel: rows staged in shared memory by bulk
    copies): random shapes with innermost 3..31 at sizes spanning many tiles and a ragged last
    tile, integer data exact and real data within 1e-12, deterministic; a p that is not 16-byte
    aligned takes the flat kernel with the same results; outer unit axes."""
    rng = np.random.default_rng(2101 if dtype == np.float32 else 2102)
    shapes = [(300, 301, 7), (7,) * 7, (5, 1, 3001, 3), (1001, 31), (13, 17, 19, 23), (2, 3, 5, 9),
              (1, 4097, 15), (64, 63, 11)]
    for sh in shapes:
        plan = T.triot_plan_describe(2, [sh], None, len(sh), 0 if dtype == np.float32 else 1, 0)
        assert plan["evrows"], sh
        for kind in ("int", "real"):
            p = (rng.integers(0, 256, size=sh).astype(dtype) if kind == "int"
                 else rng.random(sh).astype(dtype))
            ref = O.expected_value(p)
            got = T.expected_value(_dev(p)).cpu().numpy()
            if kind == "int":
                np.testing.assert_array_equal(got, ref)
            else:
                assert np.all(np.abs(got - ref) <= 1e-12 * np.abs(ref)), (sh, got, ref)
                again = T.expected_value(_dev(p)).cpu().numpy()
                np.testing.assert_array_equal(got, again)
                mis = T.expected_value(_dev(p, 1)).cpu().numpy()     # flat kernel path
                assert np.all(np.abs(mis - ref) <= 1e-12 * np.abs(ref))
            m = T.expected_value(_dev(p), with_mass=True).cpu().numpy()
            assert abs(m[-1] - math.fsum(p.astype(np.float64).ravel())) <= 1e-12 * m[-1] + 1e-300


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_ev_view_tma_tiles_vs_oracle(dtype):
    """EV of view windows with rows of 32..256 elements (TMA tensor tiles, ev_view_tma_kernel):
    window ranks 2..5 (+ unit axes folded into the map address), odd and even row lengths,
    windows ending at the base edge (TMA zero fill past it) and inside it (masked columns and
    rows) -- exact on integer data, 1e-12 on real data, deterministic."""
    rng = np.random.default_rng(3301 if dtype == np.float32 else 3302)
    cases = [((264, 264, 264), (5, 5, 5), (255, 255, 255)),
             ((40, 300), (3, 20), (37, 255)),
             ((20, 30, 256), (1, 2, 0), (19, 27, 256)),
             ((6, 7, 8, 64), (1, 0, 2, 32), (5, 7, 6, 32)),
             ((3, 4, 5, 6, 100), (1, 1, 1, 1, 4), (2, 3, 4, 5, 96)),
             ((4, 9, 1, 96), (2, 0, 0, 8), (1, 9, 1, 88)),       # unit axes in the window
             ((50, 64), (7, 0), (43, 64))]
    for base_shape, start, shape in cases:
        esz = np.dtype(dtype).itemsize
        if (base_shape[-1] * esz) % 16:
            continue
        for kind in ("int", "real"):
            base = (rng.integers(0, 256, size=base_shape).astype(dtype) if kind == "int"
                    else rng.random(base_shape).astype(dtype))
            win = base[tuple(slice(s0, s0 + w) for s0, w in zip(start, shape))].copy()
            ref = O.expected_value(win)
            tb = _dev(base)
            got = T.expected_value_view(T.View(tb, start, shape)).cpu().numpy()
            if kind == "int":
                np.testing.assert_array_equal(got, ref)
            else:
                assert np.all(np.abs(got - ref) <= 1e-12 * np.abs(ref) + 1e-300), (shape, got, ref)
                again = T.expected_value_view(T.View(tb, start, shape)).cpu().numpy()
                np.testing.assert_array_equal(got, again)
            m = T.expected_value_view(T.View(tb, start, shape), with_mass=True).cpu().numpy()
            assert abs(m[-1] - math.fsum(win.astype(np.float64).ravel())) <= 1e-12 * abs(m[-1]) + 1e-300


@pytest.mark.slow
def test_bench_partition_path_runs():
    """bench.py's multi-GPU partition path (outer-loop boxes, offset EV, NCCL all_gather,
    triot_sum_rows in rank order) end to end at world size 1 (--split-test): one JSON line with
    the step's metric -- so a one-GPU box exercises every line the N-GPU run takes."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("MASTER_ADDR", "MASTER_PORT", "RANK",
                                                             "WORLD_SIZE", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--split-test",
                        "--steps", "5", "--warmup", "3", "--no-cpu-baseline", "--no-isolated",
                        "--e2e-steps", "1"], capture_output=True, text=True, timeout=600, env=env,
                       cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["value"] > 1000 and line["gpu_launches"] == 25 and line["e2e"]["value"] > 0
    assert "NCCL process group up" in r.stderr
