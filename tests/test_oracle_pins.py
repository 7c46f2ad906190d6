"""Pins for the CPU oracle (oracle/triot_oracle.c) -- run without a GPU.

The oracle is checked against things other than itself (the task's rule ③):
  * the paper's worked example (651) and hand-derived examples (tests/golden/),
  * an independent brute-force checker: itertools.product enumeration + the explicit
    sum-of-products formula of P:50 (not Horner, not Alg 3),
  * numpy library special cases (slicing, np.pad, marginal sums),
  * closed forms (uniform 2^-24 PMF -> 7.5 exactly, separable PMFs, delta PMFs) and exact
    rational arithmetic (fractions.Fraction) on tiny shapes,
  * the exact carry count implied by P:129's amortisation argument.
Each case is chosen so that a plausible slip (a dropped term, a transposed operand, a wrong
index or sign) fails at least one test.
"""
import itertools
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import oracle as O
from triot_inputs import CONFIGS, make_inputs, random_shape, random_values, special_values

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- independent brute checker

def p50_flat_index(t, shape):
    """Explicit P:50 sum: t_0*s_1*...*s_{d-1} + t_1*s_2*...*s_{d-1} + ... + t_{d-1}."""
    d = len(shape)
    return sum(t[k] * math.prod(shape[k + 1:]) for k in range(d))


def brute_tuples(shape):
    return list(itertools.product(*[range(s) for s in shape]))


def brute_embed(dst_shape, src):
    out = np.zeros(dst_shape, dtype=src.dtype)
    of, sf = out.reshape(-1), src.reshape(-1)
    for t in brute_tuples(dst_shape):
        if all(t[k] < src.shape[k] for k in range(len(t))):
            of[p50_flat_index(t, dst_shape)] = sf[p50_flat_index(t, src.shape)]
    return out


# ---------------------------------------------------------------- golden files

def _golden_lines(name):
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                yield [part.strip() for part in line.split(";")]


def _ints(s):
    return [int(x) for x in s.split()]


def test_paper_worked_example_651():
    """(2,0,4,1) in shape (4,9,7,5) has flat index 2*9*7*5 + 0*7*5 + 4*5 + 1 = 651."""
    rows = list(_golden_lines("paper_horner_651.txt"))
    assert rows
    for shape, tup, expect in rows:
        shape, tup, expect = _ints(shape), _ints(tup), int(expect)
        assert O.tuple_to_index(tup, shape) == expect
        assert p50_flat_index(tup, shape) == expect
        assert O.index_to_tuple(expect, shape) == tuple(tup)


def test_derived_index_examples():
    n = 0
    for kind, args, expect in _golden_lines("derived_index_examples.txt"):
        parts = [_ints(a) for a in args.split("|")]
        if kind == "tuple_to_index":
            assert O.tuple_to_index(parts[0], parts[1]) == int(expect), args
        elif kind == "index_to_tuple":
            assert O.index_to_tuple(parts[0][0], parts[1]) == tuple(_ints(expect)), args
        elif kind == "advance_tuple":
            assert O.advance_tuple(parts[0], parts[1]) == tuple(_ints(expect)), args
        elif kind == "reindex":
            assert O.reindex(parts[0][0], parts[1], parts[2]) == int(expect), args
        elif kind == "reindex_powers_of_2":
            assert O.reindex_powers_of_2(parts[0][0], parts[1], parts[2]) == int(expect), args
        else:
            raise AssertionError(kind)
        n += 1
    assert n >= 10


# ---------------------------------------------------------------- L0 invariants

@pytest.mark.parametrize("d", list(range(1, 17)))
def test_enumeration_bijection_order_and_carries(d):
    """Alg 3 from the zero tuple visits every tuple once, in lexicographic order, and
    digit k (k >= 1) wraps exactly N / prod_{j>=k} s_j - 1 times (made exact)."""
    rng = np.random.default_rng(100 + d)
    shape = random_shape(rng, d, max_elems=20000, lo=1, hi=5 if d > 6 else 9)
    tuples = O.enumerate_tuples(shape)
    n = math.prod(shape)
    assert tuples.shape == (n, d)
    brute = np.array(brute_tuples(shape), dtype=np.uint64).reshape(n, d)
    np.testing.assert_array_equal(tuples, brute)
    # flat index of the i-th tuple is i, by Alg 2 and by the P:50 sum
    for i in rng.integers(0, n, size=min(n, 200)):
        t = [int(x) for x in tuples[i]]
        assert O.tuple_to_index(t, shape) == i == p50_flat_index(t, shape)
    # exact carry counts: digit k carries out at a step iff some digit left of k changes
    for k in range(1, d):
        wraps = int(np.sum(np.any(tuples[1:, :k] != tuples[:-1, :k], axis=1)))
        assert wraps == n // math.prod(shape[k:]) - 1
        # and every carry leaves digits k..d-1 at zero (Alg 3 resets them)
        changed = np.any(tuples[1:, :k] != tuples[:-1, :k], axis=1)
        assert not np.any(tuples[1:][changed][:, k:])


@pytest.mark.parametrize("d", list(range(1, 17)))
def test_index_tuple_round_trip(d):
    rng = np.random.default_rng(200 + d)
    shape = random_shape(rng, d, max_elems=10 ** 9, lo=1, hi=min(40, max(3, int(1.5 * 1e9 ** (1 / d)))))
    n = math.prod(shape)
    for i in list(rng.integers(0, n, size=64)) + [0, n - 1]:
        t = O.index_to_tuple(int(i), shape)
        assert all(0 <= t[k] < shape[k] for k in range(d))
        assert O.tuple_to_index(t, shape) == int(i) == p50_flat_index(t, shape)


def test_reindex_coherence_and_pow2():
    rng = np.random.default_rng(7)
    for d in range(1, 7):
        s = random_shape(rng, d, 5000, lo=1, hi=9)
        s2 = tuple(x + int(rng.integers(0, 4)) for x in s)
        for i in range(math.prod(s)):
            t = O.index_to_tuple(i, s)
            assert O.reindex(i, s, s2) == p50_flat_index(t, s2)
    # Alg 12 equals Alg 4 on power-of-two shapes, exhaustively on (4,8) -> (8,16)
    for i in range(32):
        assert O.reindex_powers_of_2(i, [2, 3], [3, 4]) == O.reindex(i, [4, 8], [8, 16])


# ---------------------------------------------------------------- embed

def _bits(a):
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("d", [1, 2, 3, 4, 5, 7, 10, 16])
def test_embed_vs_brute_and_numpy(dtype, d):
    rng = np.random.default_rng(300 + d)
    src_shape = random_shape(rng, d, 3000, lo=1, hi=6 if d > 5 else 12)
    # pad on some axes, crop on others
    dst_shape = tuple(max(1, s + int(rng.integers(-2, 4))) for s in src_shape)
    if math.prod(dst_shape) > 6000:
        dst_shape = tuple(min(a, b) for a, b in zip(dst_shape, src_shape))
    src = random_values(rng, src_shape, dtype, "normal")
    dst = np.full(dst_shape, np.nan, dtype=src.dtype)        # poisoned: full-write contract
    O.embed(dst, src)
    np.testing.assert_array_equal(_bits(dst), _bits(brute_embed(dst_shape, src)))
    # numpy slice idiom (the numpy listing of Alg 13)
    ref = np.zeros(dst_shape, dtype=src.dtype)
    sl = tuple(slice(0, min(a, b)) for a, b in zip(dst_shape, src_shape))
    ref[sl] = src[sl]
    np.testing.assert_array_equal(_bits(dst), _bits(ref))


def test_embed_pad_properties_C1():
    """C1: padded region is all-zero bits, src region bit-identical, exact sum preserved, and the
    result equals np.pad (pad case, src inside dst)."""
    inp = make_inputs("C1")
    src, dst_shape = inp["src"], inp["dst_shape"]
    dst = np.full(dst_shape, -1.0)
    O.embed(dst, src)
    np.testing.assert_array_equal(dst, np.pad(src, [(0, D - S) for D, S in zip(dst_shape, src.shape)]))
    sl = tuple(slice(0, s) for s in src.shape)
    np.testing.assert_array_equal(_bits(dst[sl]), _bits(src))
    mask = np.ones(dst_shape, bool)
    mask[sl] = False
    assert not np.any(_bits(dst)[mask])
    assert math.fsum(dst.ravel()) == math.fsum(src.ravel())
    assert sorted(dst[dst != 0].tolist()) == sorted(src[src != 0].tolist())


def test_embed_examples():
    # dst (2,2) from a 3x3 identity -> [[1,0],[0,1]]
    dst = np.full((2, 2), 7.0)
    O.embed(dst, np.eye(3))
    np.testing.assert_array_equal(dst, [[1, 0], [0, 1]])
    # equal shapes -> exact copy
    x = np.random.default_rng(1).random((3, 4, 5))
    y = np.empty_like(x)
    O.embed(y, x)
    np.testing.assert_array_equal(_bits(y), _bits(x))
    # empty src -> dst all +0.0; empty dst -> no-op
    dst = np.full((3, 4), np.nan)
    O.embed(dst, np.zeros((0, 4)))
    assert not np.any(_bits(dst))
    O.embed(np.zeros((0, 4)), x[:, :4, 0].copy())


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_embed_moves_raw_bits(dtype):
    sv = special_values(dtype)
    src = sv.reshape(2, 4)
    dst = np.full((3, 5), 1.0, dtype=src.dtype)
    O.embed(dst, src)
    np.testing.assert_array_equal(_bits(dst[:2, :4]), _bits(src))
    assert not np.any(_bits(dst[2, :])) and not np.any(_bits(dst[:, 4]))   # +0.0, never -0.0


def test_embed_crop_is_benchmark1_body():
    """Benchmark 1: x[t] = y[t] over x's (smaller) shape.  Scaled down
    copy of (2^10,2^9,2^8) -> (2^9,2^9,2^5), ratios kept."""
    y = np.random.default_rng(11).random((64, 32, 16))
    x = np.empty((32, 32, 2))
    O.embed(x, y)
    np.testing.assert_array_equal(x, y[:32, :32, :2])


def test_embed_region_only():
    rng = np.random.default_rng(12)
    src = rng.random((3, 5, 2))
    dst = np.full((4, 3, 6), 9.0)
    O.embed(dst, src, region_only=True)
    ref = np.full((4, 3, 6), 9.0)
    ref[:3, :3, :2] = src[:3, :3, :2]
    np.testing.assert_array_equal(dst, ref)


# ---------------------------------------------------------------- binary

@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("op", ["add", "sub", "mul", "div"])
@pytest.mark.parametrize("d", [1, 2, 3, 5, 8, 16])
def test_binary_vs_numpy_slices(dtype, op, d):
    rng = np.random.default_rng(400 + d)
    ish = random_shape(rng, d, 2000, lo=1, hi=5 if d > 5 else 10)
    a = random_values(rng, tuple(s + int(rng.integers(0, 3)) for s in ish), dtype, "normal")
    b = random_values(rng, tuple(s + int(rng.integers(0, 3)) for s in ish), dtype, "normal")
    c = O.apply_binary(a, b, op, iter_shape=ish)
    sl = tuple(slice(0, s) for s in ish)
    fn = {"add": np.add, "sub": np.subtract, "mul": np.multiply, "div": np.divide}[op]
    with np.errstate(all="ignore"):
        ref = fn(a[sl], b[sl])
    np.testing.assert_array_equal(_bits(c), _bits(np.ascontiguousarray(ref)))


def test_binary_closed_forms():
    rng = np.random.default_rng(13)
    a = rng.random((5, 7, 3))
    ones = np.ones((6, 4, 3))
    c = O.apply_binary(a, ones, "mul")                  # B == 1 -> crop(A) bitwise
    np.testing.assert_array_equal(_bits(c), _bits(np.ascontiguousarray(a[:5, :4, :3])))
    b = rng.random((6, 4, 3))
    np.testing.assert_array_equal(O.apply_binary(a, b, "mul"), O.apply_binary(b, a, "mul"))
    np.testing.assert_array_equal(O.apply_binary(a, b, "add"), O.apply_binary(b, a, "add"))
    # c larger than iter: elements outside iter are untouched
    out = np.full((7, 5, 4), -3.0)
    O.apply_binary(a, b, "sub", iter_shape=(5, 4, 3), out=out)
    np.testing.assert_array_equal(out[:5, :4, :3], a[:5, :4, :3] - b[:5, :4, :3])
    assert np.all(out[5:] == -3.0) and np.all(out[:, 4:] == -3.0) and np.all(out[:, :, 3:] == -3.0)


def test_binary_C4_sampled():
    """C4 at full size is 25 M tuples; check a slab against numpy."""
    inp = make_inputs("C4")
    a, b = inp["a"][:2].copy(), inp["b"][:2].copy()
    ish = (2,) + inp["iter_shape"][1:]
    c = O.apply_binary(a, b, "mul", iter_shape=ish)
    np.testing.assert_array_equal(c, a[:, :32, :24, :32, :32] * b[:, :32, :24, :32, :32])


# ---------------------------------------------------------------- expected value

def test_ev_uniform_exact_7_5():
    """Uniform PMF over (16)^6 with p = 2^-24: every partial sum is exact, so E[t_k] = 7.5."""
    p = np.full((16,) * 6, 2.0 ** -24)
    m, plain = O.expected_value(p, with_plain=True)
    assert list(m) == [7.5] * 6 and list(plain) == [7.5] * 6


def test_ev_separable_closed_form():
    rng = np.random.default_rng(14)
    shape = (5, 3, 7, 4)
    qs = []
    for s in shape:
        q = rng.random(s)
        qs.append(q / q.sum())
    p = qs[0]
    for q in qs[1:]:
        p = np.multiply.outer(p, q)
    m = O.expected_value(np.ascontiguousarray(p))
    for k, q in enumerate(qs):
        expect = math.fsum(v * q[v] for v in range(len(q))) * math.fsum(p.ravel())
        assert abs(m[k] - expect) <= 1e-13 * abs(expect)


def test_ev_delta():
    p = np.zeros((4, 6, 3, 5))
    p[3, 1, 2, 4] = 1.0
    assert list(O.expected_value(p)) == [3.0, 1.0, 2.0, 4.0]


def test_ev_integer_valued_exact_vs_brute():
    rng = np.random.default_rng(15)
    for d in (1, 2, 3, 5):
        shape = random_shape(rng, d, 3000, lo=1, hi=9)
        p = rng.integers(0, 256, size=shape).astype(np.float64)
        m = O.expected_value(p)
        pf = p.ravel()
        for k in range(d):
            exact = sum(t[k] * int(pf[p50_flat_index(t, shape)]) for t in brute_tuples(shape))
            assert m[k] == float(exact)


def test_ev_fraction_brute_force():
    rng = np.random.default_rng(16)
    for d in (2, 3, 4):
        shape = random_shape(rng, d, 400, lo=1, hi=7)
        p = rng.random(shape)
        m = O.expected_value(p)
        pf = p.ravel()
        for k in range(d):
            exact = sum(Fraction(t[k]) * Fraction(float(pf[p50_flat_index(t, shape)]))
                        for t in brute_tuples(shape))
            assert abs(Fraction(m[k]) - exact) <= Fraction(1, 10 ** 15) * max(abs(exact), 1)


def test_ev_abs_scale_fraction_brute_force():
    """oracle_expected_value_abs = sum_t |t_k * p[t]| (the scale of SURVEY Q12's signed-input
    bound on Alg 11's terms), against itertools + the P:50 sum in exact rationals, on
    signed inputs (a dropped abs, a dropped t_k weight or a wrong index fails), f64 and f32."""
    rng = np.random.default_rng(161)
    for d in (1, 2, 3, 4, 5):
        for dt in (np.float64, np.float32):
            shape = random_shape(rng, d, 500, lo=1, hi=7)
            p = (rng.standard_normal(shape) * 3.0).astype(dt)
            got = O.expected_value_abs(p)
            pf = p.ravel()
            for k in range(d):
                exact = sum(abs(Fraction(t[k]) * Fraction(float(pf[p50_flat_index(t, shape)])))
                            for t in brute_tuples(shape))
                # a sum of <= 500 non-negative terms, each rounded once: rel error <= 1e-13
                assert abs(Fraction(got[k]) - exact) <= Fraction(1, 10 ** 13) * max(exact, 1e-300)


def test_ev_abs_scale_closed_form_minus_one():
    """p == -1 everywhere: sum_t |t_k * p[t]| = sum_t t_k = N * (n_k - 1) / 2, an exact integer."""
    for shape in [(5,), (3, 4), (2, 7, 3), (4, 1, 6, 2), (3, 3, 3, 3, 3)]:
        for dt in (np.float64, np.float32):
            p = np.full(shape, -1.0, dtype=dt)
            got = O.expected_value_abs(p)
            n = math.prod(shape)
            assert list(got) == [float(n * (s - 1) // 2) for s in shape], (shape, got)
            # and the signed sum is its negation (same terms, sign flipped)
            assert list(O.expected_value(p)) == [-float(n * (s - 1) // 2) for s in shape]


def test_ev_abs_scale_equals_ev_on_nonnegative_input():
    """On p >= 0 every term t_k p[t] is non-negative, so the scale equals the integer-exact EV."""
    rng = np.random.default_rng(162)
    p = rng.integers(0, 256, size=(6, 5, 7, 4)).astype(np.float64)
    assert list(O.expected_value_abs(p)) == list(O.expected_value(p))


def test_ev_numpy_marginal_route_C3():
    """'marginalization': E[t_k] = sum_v v * (sum of p over axes != k)[v]."""
    p = make_inputs("C3")["p"]
    m = O.expected_value(p)
    for k in range(6):
        axes = tuple(j for j in range(6) if j != k)
        marg = p.sum(axis=axes)
        ref = math.fsum(v * marg[v] for v in range(16))
        assert abs(m[k] - ref) <= 1e-13 * ref
        assert 7.49 < m[k] < 7.51


def test_ev_f32_input_widened():
    rng = np.random.default_rng(17)
    p32 = rng.random((6, 5, 4)).astype(np.float32)
    np.testing.assert_array_equal(O.expected_value(p32), O.expected_value(p32.astype(np.float64)))


def test_configs_table_matches_baseline_json():
    import json
    with open(os.path.join(os.path.dirname(GOLDEN), "..", "BASELINE.json")) as f:
        base = json.load(f)
    text = " ".join(base["configs"])
    for c in CONFIGS.values():
        for shp in c.shapes.values():
            if len(set(shp)) == 1 and len(shp) > 4:
                continue
            assert str(shp).replace(" ", "").replace(",)", ")") in text.replace(" ", ""), (c.name, shp)


# ---------------------------------------------------------------- NEXT-1: views

def test_view_bias_and_visits_spec_example():
    """P:605 bias; a (2,2) window at (1,2) of a (4,5) base has bias 7 and visits base
    flat indices {7, 8, 12, 13}."""
    assert O.view_bias([1, 2], [4, 5]) == 7
    base = np.arange(20, dtype=np.float64).reshape(4, 5)
    out = np.zeros((2, 2))
    # embed from the view into a dense (2,2): the view's elements in order
    O.embed_view(out, [0, 0], [2, 2], base, [1, 2], [2, 2])
    assert out.ravel().tolist() == [7.0, 8.0, 12.0, 13.0]


@pytest.mark.parametrize("seed", range(8))
def test_views_are_transparent(seed):
    """any op on a view equals the op on a materialised copy of the window (numpy slice)."""
    rng = np.random.default_rng(600 + seed)
    d = int(rng.integers(1, 6))
    base_a = rng.standard_normal(random_shape(rng, d, 4000, lo=2, hi=9))
    win = tuple(int(rng.integers(1, s + 1)) for s in base_a.shape)
    start_a = tuple(int(rng.integers(0, s - w + 1)) for s, w in zip(base_a.shape, win))
    base_b = rng.standard_normal(tuple(w + int(rng.integers(0, 4)) for w in win))
    start_b = tuple(int(rng.integers(0, s - w + 1)) for s, w in zip(base_b.shape, win))
    base_c = np.full(tuple(w + int(rng.integers(0, 3)) for w in win), 7.0)
    start_c = tuple(int(rng.integers(0, s - w + 1)) for s, w in zip(base_c.shape, win))
    sl = lambda st, w: tuple(slice(a, a + b) for a, b in zip(st, w))
    mat_a, mat_b = base_a[sl(start_a, win)].copy(), base_b[sl(start_b, win)].copy()
    # binary on views == binary on copies; c outside its window untouched
    ref_c = base_c.copy()
    ref_c[sl(start_c, win)] = mat_a * mat_b
    O.apply_binary_view(base_c, start_c, base_a, start_a, base_b, start_b, win, "mul")
    np.testing.assert_array_equal(base_c, ref_c)
    # embed view -> view, pad and crop: == embed on the materialised windows
    dwin = tuple(max(1, w + int(rng.integers(-1, 3))) for w in win)
    dbase = np.full(tuple(w + 2 for w in dwin), -1.0)
    dstart = (1,) * d
    ref_d = dbase.copy()
    tmp = np.empty(dwin)
    O.embed(tmp, mat_a)
    ref_d[sl(dstart, dwin)] = tmp
    O.embed_view(dbase, dstart, dwin, base_a, start_a, win)
    np.testing.assert_array_equal(dbase, ref_d)


def test_pmf_product_over_intersecting_support():
    """two PMFs over supports with different origins; views window the intersection.
    A has support rows 2..6, cols 0..4; B has rows 4..8, cols 1..3.  The product over the
    intersection (rows 4..5, cols 1..3) equals the numpy product of the aligned slices."""
    rng = np.random.default_rng(77)
    A = rng.random((5, 5)); A /= A.sum()       # support origin (2, 0)
    B = rng.random((5, 3)); B /= B.sum()       # support origin (4, 1)
    lo = (4, 1); hi = (min(2 + 5, 4 + 5), min(0 + 5, 1 + 3))
    win = (hi[0] - lo[0], hi[1] - lo[1])
    a_start = (lo[0] - 2, lo[1] - 0)
    b_start = (lo[0] - 4, lo[1] - 1)
    C = np.zeros(win)
    O.apply_binary_view(C, (0, 0), A, a_start, B, b_start, win, "mul")
    ref = A[2:2 + win[0], 1:1 + win[1]] * B[0:win[0], 0:win[1]]
    np.testing.assert_array_equal(C, ref)


# ---------------------------------------------------------------- NEXT-2: Benchmark 2 inner product

def test_inner_product_examples():
    """x = [[1,2],[3,4]], y = 3x3 identity, over (2,2) -> 5."""
    x = np.array([[1.0, 2.0], [3.0, 4.0]])
    assert O.inner_product(x, np.eye(3)) == 5.0
    assert O.inner_product(x, np.zeros((3, 3))) == 0.0


def test_inner_product_exact_and_numpy():
    rng = np.random.default_rng(31)
    for d in (1, 2, 3, 5):
        sa = random_shape(rng, d, 2000, lo=1, hi=9)
        sb = tuple(s + int(rng.integers(-1, 3)) if s > 1 else s for s in sa)
        a = rng.integers(-100, 100, size=sa).astype(np.float64)
        b = rng.integers(-100, 100, size=sb).astype(np.float64)
        ish = tuple(min(x, y) for x, y in zip(sa, sb))
        sl = tuple(slice(0, m) for m in ish)
        exact = int(np.sum(a[sl].astype(np.int64) * b[sl].astype(np.int64)))
        assert O.inner_product(a, b) == float(exact)
    # real values: within 1e-15 of the exact rational sum (tiny) and of numpy (1e-13)
    a = rng.standard_normal((3, 4, 5)); b = rng.standard_normal((4, 4, 6))
    ish = (3, 4, 5)
    exact = sum(Fraction(float(a[t])) * Fraction(float(b[t])) for t in brute_tuples(ish))
    got = O.inner_product(a, b)
    scale = sum(abs(Fraction(float(a[t])) * Fraction(float(b[t]))) for t in brute_tuples(ish))
    # each product is rounded once (rel 2^-53); the compensated sum adds no more than that
    assert abs(Fraction(got) - exact) <= Fraction(1, 10 ** 15) * scale
    big_a = rng.standard_normal((64, 32, 16)); big_b = rng.standard_normal((32, 32, 8))
    ref = float(np.dot(big_a[:32, :32, :8].ravel(), big_b.ravel()))
    assert abs(O.inner_product(big_a, big_b) - ref) <= 1e-12 * np.sum(np.abs(big_a[:32, :32, :8] * big_b))


# ---------------------------------------------------------------- NEXT-3: Benchmark 3 fused update

def test_fused_update_examples():
    """x=[2], y=[3], z=[1] -> 2 + 3*2 - 1 = 7; y = z = 0 leaves x unchanged."""
    x = np.array([2.0]); O.fused_update(x, np.array([3.0]), np.array([1.0]))
    assert x.tolist() == [7.0]
    x = np.random.default_rng(1).random((3, 4)); x0 = x.copy()
    O.fused_update(x, np.zeros((5, 5)), np.zeros((3, 4)))
    np.testing.assert_array_equal(x, x0)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_fused_update_vs_numpy(dtype):
    """numpy evaluates (x + (y*x)) - z with one rounding per operation, like C with contraction
    off: bit-exact on the paper's Benchmark-3 shape family (scaled down)."""
    rng = np.random.default_rng(32)
    x = random_values(rng, (9, 4, 13, 6), dtype, "normal")
    y = random_values(rng, (12, 8, 15, 7), dtype, "normal")
    z = random_values(rng, (10, 5, 16, 9), dtype, "normal")
    sl = tuple(slice(0, s) for s in x.shape)
    ref = (x + (y[sl] * x)) - z[sl]
    got = x.copy()
    O.fused_update(got, y, z)
    np.testing.assert_array_equal(_bits(got), _bits(ref))


# ---------------------------------------------------------------- NEXT-4: naive convolution (Alg 15)

def test_convolve_examples():
    """[1,2] * [3,4] = [3,10,8]; a unit impulse is the identity; [[1,1],[1,1]] * [[1]]."""
    assert O.naive_convolve(np.array([1.0, 2.0]), np.array([3.0, 4.0])).tolist() == [3.0, 10.0, 8.0]
    x = np.random.default_rng(2).random((3, 4, 2))
    np.testing.assert_array_equal(O.naive_convolve(x, np.ones((1, 1, 1))), x)
    np.testing.assert_array_equal(O.naive_convolve(np.ones((2, 2)), np.ones((1, 1))), np.ones((2, 2)))


def test_convolve_vs_scipy_and_conservation():
    import scipy.signal
    rng = np.random.default_rng(41)
    for d in (1, 2, 3):
        ls = random_shape(rng, d, 300, lo=1, hi=9)
        rs = random_shape(rng, d, 300, lo=1, hi=9)
        li = rng.integers(-20, 20, size=ls).astype(np.float64)
        ri = rng.integers(-20, 20, size=rs).astype(np.float64)
        ref = scipy.signal.convolve(li, ri, method="direct")
        np.testing.assert_array_equal(O.naive_convolve(li, ri), ref)          # integers: exact
        lf, rf = rng.random(ls), rng.random(rs)
        got = O.naive_convolve(lf, rf)
        np.testing.assert_allclose(got, scipy.signal.convolve(lf, rf, method="direct"),
                                   rtol=1e-13, atol=0)
        assert abs(math.fsum(got.ravel()) - math.fsum(lf.ravel()) * math.fsum(rf.ravel())) <= \
            1e-12 * math.fsum(got.ravel())
    # f32: same recurrence in float
    lf = rng.random((5, 3)).astype(np.float32); rf = rng.random((4, 2)).astype(np.float32)
    got = O.naive_convolve(lf, rf)
    assert got.dtype == np.float32 and got.shape == (8, 4)
    np.testing.assert_allclose(got, scipy.signal.convolve(lf.astype(np.float64),
                                                          rf.astype(np.float64)), rtol=1e-5)


def test_convolve_order_is_lhs_lexicographic():
    """Alg 15 adds the contributions to one output in lexicographic order of the lhs tuple
    (the outer enumerate): reproduce that order with an explicit Python sum and compare bits."""
    rng = np.random.default_rng(42)
    lhs, rhs = rng.standard_normal((4, 3)), rng.standard_normal((3, 2))
    got = O.naive_convolve(lhs, rhs)
    for u in brute_tuples(got.shape):
        acc = 0.0
        for tl in brute_tuples(lhs.shape):
            tr = tuple(a - b for a, b in zip(u, tl))
            if all(0 <= tr[k] < rhs.shape[k] for k in range(2)):
                acc = acc + lhs[tl] * rhs[tr]
        assert got[u] == acc
