"""The C-ABI boundary without a GPU: the library loads, exports every symbol include/triot.h
declares, validates exactly as the header states, and its host plan (canonicalisation, vector
geometry, carry deltas, fast-division magics) is checked against the oracle through a CPU model
of the kernel algorithm (tests/kernel_model.py).  No compute call reaches the device here."""
import ctypes
import math
import os
import re
import subprocess

import numpy as np
import pytest

from oracle import oracle as O
from triot_inputs import CONFIGS, random_shape, random_values
from tests import kernel_model

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "triot.h")

T = pytest.importorskip("paper_1608_00099_b200")
L = T._lib

F32, F64 = L.TRIOT_F32, L.TRIOT_F64
FAKE = 1 << 40        # a 256-byte-aligned fake device address; validation never dereferences


def declared_symbols():
    with open(HEADER) as f:
        text = f.read()
    return sorted(set(re.findall(r"TRIOT_API\s+[\w\s\*]+?\b(triot_\w+)\s*\(", text)))


def test_exports_every_declared_symbol():
    decl = declared_symbols()
    assert len(decl) == 23, decl
    out = subprocess.run(["nm", "-D", "--defined-only", T.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = sorted(set(re.findall(r"\bT (triot_\w+)", out)))
    assert exported == decl
    assert tuple(sorted(L.EXPORTS)) == tuple(decl)
    lib = ctypes.CDLL(T.LIB_PATH)
    for name in decl:
        assert getattr(lib, name)


def test_no_torch_or_oracle_linkage():
    out = subprocess.run(["ldd", T.LIB_PATH], capture_output=True, text=True).stdout
    assert "torch" not in out and "oracle" not in out and "libcudart" not in out


def test_constants_and_status_strings():
    assert T.triot_max_dimension() == 16
    for code, name in L.STATUS.items():
        assert T.triot_status_string(code) == name


def test_launch_policy_range():
    """Modes -1..5 and 0..1024 blocks per SM are accepted (host state only); others rejected."""
    lib = L.lib()
    try:
        for mode in range(-1, 6):
            assert lib.triot_set_launch_policy(mode, 16) == 0
        for mode, bpsm in [(-2, 0), (6, 0), (0, -1), (0, 1025)]:
            assert lib.triot_set_launch_policy(mode, bpsm) == 5
            assert "BadPolicy" in T.triot_last_error()
    finally:
        lib.triot_set_launch_policy(-1, 0)


def _embed(dst_shape, src_shape, d=None, dtype=F64, flags=0, dst=FAKE, src=FAKE * 2):
    d = len(dst_shape) if d is None else d
    return T.triot_embed(dst, dst_shape, src, src_shape, d, dtype, flags, 0)


def test_validation_embed():
    ok_cuda = L.STATUS[9]
    assert _embed((2, 2), (2, 2), d=0) == 2
    assert _embed((2,) * 17, (2,) * 17) == 2
    assert "d = 17" in T.triot_last_error()
    assert _embed((2, -1), (2, 2)) == 3
    assert "axis 1" in T.triot_last_error()
    assert _embed((1 << 31, 1 << 31), (2, 2)) == 3          # >= 2^62 bytes
    assert _embed((2, 2), (2, 2), dtype=7) == 5
    assert _embed((2, 2), (2, 2), flags=4) == 5
    assert _embed((2, 2), (2, 2), dst=0) == 1
    assert _embed((2, 2), (2, 2), src=0) == 1
    assert _embed((2, 2), (2, 2), dst=FAKE + 4) == 6          # f64 needs 8-byte alignment
    assert _embed((4, 4), (4, 4), src=FAKE + 64) == 7         # overlap
    # empty dst: a no-op that touches nothing, so NULL pointers are fine
    assert _embed((0, 4), (3, 4), dst=0, src=0) == 0
    assert T.triot_embed(FAKE, None, FAKE * 2, (2, 2), 2, F64, 0, 0) == 1
    del ok_cuda


def test_validation_binary_check_bounds():
    # iter (3,3) over (2,3) -> AxisOutOfBounds(tensor 0, axis 0)
    st = T.triot_apply_binary(FAKE, None, FAKE * 2, (2, 3), FAKE * 3, (3, 3), (3, 3), 2, F64,
                              L.TRIOT_MUL, 0)
    assert st == 4
    msg = T.triot_last_error()
    assert "'a'" in msg and "axis 0" in msg
    st = T.triot_apply_binary(FAKE, (2, 2), FAKE * 2, (3, 3), FAKE * 3, (3, 3), (2, 3), 2, F64,
                              L.TRIOT_MUL, 0)
    assert st == 4 and "'c'" in T.triot_last_error() and "axis 1" in T.triot_last_error()
    assert T.triot_apply_binary(FAKE, None, FAKE * 2, (2, 2), FAKE * 3, (2, 2), None, 2, F64, 9,
                                0) == 5
    # aliasing: c overlapping a with different shapes is refused, exact in-place is allowed
    assert T.triot_apply_binary(FAKE, (4, 4), FAKE + 8, (4, 4), FAKE * 3, (4, 4), None, 2, F64,
                                L.TRIOT_ADD, 0) == 7
    assert T.triot_apply_binary(FAKE, (4, 4), FAKE, (4, 5), FAKE * 3, (4, 4), None, 2, F64,
                                L.TRIOT_ADD, 0) == 7
    # empty iteration: no-op
    assert T.triot_apply_binary(0, None, 0, (0, 3), 0, (2, 3), None, 2, F64, L.TRIOT_ADD, 0) == 0


def test_validation_ev():
    assert T.triot_expected_value_workspace_size((16,) * 6, 6, F64) > 256
    with pytest.raises(T.TriotError):
        T.triot_expected_value_workspace_size((2,) * 17, 17, F64)
    ws = T.triot_expected_value_workspace_size((4, 4), 2, F64)
    assert T.triot_expected_value(0, FAKE, (4, 4), 2, F64, FAKE * 3, ws, 0) == 1
    assert T.triot_expected_value(FAKE + 4, FAKE * 2, (4, 4), 2, F64, FAKE * 3, ws, 0) == 6
    assert T.triot_expected_value(FAKE + 8, FAKE, (4, 4), 2, F64, FAKE * 3, ws, 0) == 7


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="GPU present")
def test_valid_call_without_gpu_reports_cuda_error():
    st = _embed((4, 4), (2, 2))
    assert st == 9 and "CUDA" in T.triot_last_error()


# ------------------------------------------------------------------ fast division magics

def _fastdiv(n, m, s):
    h = (n * m) >> 32
    return (h + ((n - h) >> (s & 0xFF))) >> (s >> 8)


def test_fastdiv_exact():
    rng = np.random.default_rng(3)
    divisors = {1, 2, 3, 4, 5, 7, 8, 9, 16, 24, 32, 36, 40, 48, 64, 384, 512, 6, 12, 2 ** 31 - 1,
                2 ** 31, 2 ** 31 + 1, 2 ** 32 - 1, 65537, 1000003}
    divisors |= set(int(x) for x in rng.integers(1, 2 ** 32, size=40))
    edge = [0, 1, 2, 3, 2 ** 16, 2 ** 31 - 1, 2 ** 31, 2 ** 32 - 2, 2 ** 32 - 1]
    for dv in sorted(divisors):
        m, s = T.triot_fastdiv_magic(dv)
        ns = edge + [int(x) for x in rng.integers(0, 2 ** 32, size=2000)]
        ns += [k * dv + r for k in (1, 2, 3, 1000) for r in (0, dv - 1) if k * dv + r < 2 ** 32]
        for n in ns:
            assert _fastdiv(n, m, s) == n // dv, (dv, n)
        if dv & (dv - 1) == 0:          # 2^k: the magic degenerates to Alg 12's shift
            assert all(_fastdiv(n, m, s) == n >> (dv.bit_length() - 1) for n in ns)
    with pytest.raises(T.TriotError):
        T.triot_fastdiv_magic(0)


# ------------------------------------------------------------------ plans of C1..C5

def _plan(name, mods=(0, 0, 0)):
    c = CONFIGS[name]
    sh = c.shapes
    dt = F32 if c.dtype == "f32" else F64
    if c.op == "embed":
        return T.triot_plan_describe(0, [sh["dst"], sh["src"]], None, len(sh["dst"]), dt, 0, mods)
    if c.op == "binary":
        return T.triot_plan_describe(1, [None, sh["a"], sh["b"]], sh["iter"], len(sh["a"]), dt,
                                     L.TRIOT_MUL, mods)
    return T.triot_plan_describe(2, [sh["p"]], None, len(sh["p"]), dt, 0, mods)


def test_plans_of_the_five_configs():
    p = _plan("C1")     # dst rows 64 B -> 32-B stores; src rows 40 B -> element loads
    assert (p["Dc"], p["D"], p["V"], p["collapsed"]) == (4, 4, 4, False)
    assert [t["vec"] for t in p["t"]] == [True, False]
    p = _plan("C2")     # both rows 32-B multiples, src/zero boundary at 1536 B is vector-aligned
    assert (p["Dc"], p["D"], p["V"]) == (3, 3, 8)
    assert [t["vec"] for t in p["t"]] == [True, True]
    assert (p["vfull"], p["vany"]) == (48, 48)
    p = _plan("C3")
    assert (p["Dc"], p["D"], p["V"]) == (6, 6, 4) and p["t"][0]["vec"]
    p = _plan("C4")     # A rows 288 B = 9 x 32 B stay aligned
    assert (p["Dc"], p["D"], p["V"]) == (5, 5, 4)
    assert [t["vec"] for t in p["t"]] == [True, True, True]
    p = _plan("C5")     # innermost 4 floats < a vector: 2 dst rows per 32-B vector
    assert (p["Dc"], p["D"], p["V"], p["R"], p["collapsed"]) == (14, 13, 8, 2, True)
    assert [t["vec"] for t in p["t"]] == [True, False]
    assert all(not pl["idx64"] for pl in map(_plan, CONFIGS))
    # misaligned output pointer: 32-B vectors stored shifted to the 32-byte grid
    p = _plan("C2", mods=(4, 0, 0))
    assert p["dshift"] == 1 and p["V"] == 8 and not p["rows"]


def test_canonicalisation_drops_and_merges():
    # equal inner extents merge (P:609 style simplification); unit axes are dropped
    p = T.triot_plan_describe(0, [(6, 1, 5, 8), (4, 1, 5, 8)], None, 4, F32, 0)
    assert p["Dc"] == 1 and p["cn"] == [240] and p["scols"] == 160   # t < 160 <=> t0 < 4
    p = T.triot_plan_describe(0, [(6, 5, 8), (4, 3, 8)], None, 3, F32, 0)
    assert p["Dc"] == 2 and p["cn"] == [6, 40]        # src row stride 24 != 40: no outer merge
    p = T.triot_plan_describe(1, [None, (3, 4, 5), (3, 4, 5)], None, 3, F64, 0)
    assert p["Dc"] == 1 and p["cn"] == [60]
    # expected value never merges: every digit is a weight (Alg 11)
    p = T.triot_plan_describe(2, [(3, 4, 5)], None, 3, F64, 0)
    assert p["Dc"] == 3


# ------------------------------------------------------------------ kernel model vs oracle

def _bits(a):
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("seed", range(12))
def test_model_embed_vs_oracle(dtype, seed):
    rng = np.random.default_rng(1000 + seed)
    d = int(rng.integers(1, 9))
    src_shape = random_shape(rng, d, 1500, lo=1, hi=7 if d > 3 else 14)
    dst_shape = tuple(max(1, s + int(rng.integers(-2, 5))) for s in src_shape)
    if seed % 4 == 0:   # tiny innermost extents -> collapsed vectors
        dst_shape = dst_shape[:-1] + (int(rng.choice([1, 2, 4])),)
    if math.prod(dst_shape) > 4000:
        dst_shape = tuple(min(a, b) for a, b in zip(dst_shape, src_shape))
    region = seed % 5 == 4
    src = random_values(rng, src_shape, dtype, "normal")
    ref = np.full(dst_shape, -7.0, dtype=src.dtype)
    O.embed(ref, src, region_only=region)
    dt = F32 if dtype == "f32" else F64
    desc = T.triot_plan_describe(0, [dst_shape, src_shape], None, d, dt, 1 if region else 0,
                                 mode=seed % 2, warps=int(rng.integers(1, 9)))
    out = np.full(dst_shape, -7.0, dtype=src.dtype)
    kernel_model.run(desc, "embed", [out.reshape(-1), src.reshape(-1)])
    np.testing.assert_array_equal(_bits(out), _bits(ref))


@pytest.mark.parametrize("dst_shape,src_shape,dtype,warps", [
    ((4,) * 7, (3,) * 7, "f32", 5),               # C5's structure at 4^7: 32 vectors = 4^2 x 2
    ((4,) * 7, (3,) * 7, "f32", 1),
    ((5, 4, 4, 2, 8), (2, 3, 4, 2, 5), "f32", 3),  # 32 vectors = 4 x 4 x 2 rows of 8
    ((3, 6, 2, 4, 4, 4), (3, 4, 1, 3, 2, 4), "f64", 7),  # f64: 4 per vector, 2 x 4 x 4 = 32
    ((4, 4, 4, 4, 4), (4, 4, 4, 4, 4), "f32", 2),  # no zeros at all
])
def test_model_embed_zero_runs_vs_oracle(dst_shape, src_shape, dtype, warps):
    """Embed zero runs (the warp stores zeros while an outer digit is out of bounds, then
    re-decodes): the plan enables them for these shapes and the model's output is the oracle's."""
    rng = np.random.default_rng(77)
    src = random_values(rng, src_shape, dtype, "normal")
    dt = F32 if dtype == "f32" else F64
    for region in (False, True):
        ref = np.full(dst_shape, -7.0, dtype=src.dtype)
        O.embed(ref, src, region_only=region)
        desc = T.triot_plan_describe(0, [dst_shape, src_shape], None, len(dst_shape), dt,
                                     1 if region else 0, mode=0, warps=warps)
        if not region and dst_shape != src_shape:
            assert desc["zmask"] != 0, desc
        out = np.full(dst_shape, -7.0, dtype=src.dtype)
        kernel_model.run(desc, "embed", [out.reshape(-1), src.reshape(-1)])
        np.testing.assert_array_equal(_bits(out), _bits(ref))


@pytest.mark.parametrize("seed", range(10))
def test_model_binary_vs_oracle(seed):
    rng = np.random.default_rng(2000 + seed)
    d = int(rng.integers(1, 8))
    dtype = "f32" if seed % 2 else "f64"
    ish = random_shape(rng, d, 1500, lo=1, hi=7 if d > 3 else 14)
    a = random_values(rng, tuple(s + int(rng.integers(0, 3)) for s in ish), dtype, "normal")
    b = random_values(rng, tuple(s + int(rng.integers(0, 3)) for s in ish), dtype, "normal")
    cs = tuple(s + int(rng.integers(0, 2)) for s in ish) if seed % 3 == 0 else ish
    op = ["add", "sub", "mul", "div"][seed % 4]
    ref = np.full(cs, 5.0, dtype=a.dtype)
    O.apply_binary(a, b, op, iter_shape=ish, out=ref)
    dt = F32 if dtype == "f32" else F64
    desc = T.triot_plan_describe(1, [cs, a.shape, b.shape], ish, d, dt, T.OPS[op],
                                 mode=seed % 2, warps=int(rng.integers(1, 9)))
    out = np.full(cs, 5.0, dtype=a.dtype)
    kernel_model.run(desc, "binary", [out.reshape(-1), a.reshape(-1), b.reshape(-1)], binop=op)
    np.testing.assert_array_equal(_bits(out), _bits(ref))


@pytest.mark.parametrize("seed", range(10))
def test_model_ev_vs_oracle(seed):
    rng = np.random.default_rng(3000 + seed)
    d = int(rng.integers(1, 8))
    shape = random_shape(rng, d, 1500, lo=1, hi=7 if d > 3 else 14)
    if seed % 3 == 0:
        shape = shape[:-1] + (int(rng.choice([1, 2, 4])),)
    p = rng.integers(0, 256, size=shape).astype(np.float64)     # exact: any order agrees
    desc = T.triot_plan_describe(2, [shape], None, d, F64, 0, mode=seed % 3,
                                 warps=int(rng.integers(1, 9)))
    got = kernel_model.run(desc, "ev", [p.reshape(-1)])
    np.testing.assert_array_equal(np.array(got), O.expected_value(p))


def test_view_validation():
    L_ = T._lib
    base = (4, 5)
    ok_dst, k1 = L_.make_view(FAKE, (8, 8), (1, 1), (4, 5))
    bad, k2 = L_.make_view(FAKE * 2, base, (1, 2), (4, 3))      # 1 + 4 > 4 on axis 0
    st = T.triot_embed_view(ok_dst, bad, 2, F64, 0, 0)
    assert st == 4 and "view 'src' axis 0" in T.triot_last_error()
    neg, k3 = L_.make_view(FAKE * 2, base, (-1, 0), (2, 2))
    assert T.triot_embed_view(ok_dst, neg, 2, F64, 0, 0) == 4
    # overlapping windows of one base are refused (conservative byte-span check)
    v1, k4 = L_.make_view(FAKE, (8, 8), (0, 0), (4, 4))
    v2, k5 = L_.make_view(FAKE, (8, 8), (2, 2), (4, 4))
    assert T.triot_embed_view(v1, v2, 2, F64, 0, 0) == 7
    # identical view in place is allowed for binary (validation passes; CPU then fails in CUDA)
    st = T.triot_apply_binary_view(v1, v1, v2, None, 2, F64, 0, 0)
    assert st == 7                                                 # c overlaps b
    del k1, k2, k3, k4, k5


def test_ev_view_validation():
    L_ = T._lib
    good, k1 = L_.make_view(FAKE, (8, 9), (1, 2), (4, 5))
    bad, k2 = L_.make_view(FAKE, (8, 9), (5, 2), (4, 5))           # 5 + 4 > 8 on axis 0
    ws = FAKE * 3
    st = T.triot_expected_value_view(FAKE * 2, bad, 2, F64, 0, ws, 1 << 20, 0)
    assert st == 4 and "view 'p' axis 0" in T.triot_last_error()
    # means inside the view's base buffer (not just its window) is refused
    st = T.triot_expected_value_view(FAKE + 8, good, 2, F64, 0, ws, 1 << 20, 0)
    assert st == 7
    assert T.triot_expected_value_view(FAKE * 2 + 4, good, 2, F64, 0, ws, 1 << 20, 0) == 6
    assert T.triot_expected_value_view(FAKE * 2, good, 2, 7, 0, ws, 1 << 20, 0) == 5
    # a valid call reaches the launch, which fails without a GPU
    assert T.triot_expected_value_view(FAKE * 2, good, 2, F64, 1, ws, 1 << 20, 0) == 9
    del k1, k2


@pytest.mark.parametrize("seed", range(6))
def test_model_views_vs_oracle(seed):
    """The host plan for views (biased pointer + base strides) run through the kernel model."""
    rng = np.random.default_rng(4000 + seed)
    d = int(rng.integers(1, 5))
    base_a = rng.standard_normal(random_shape(rng, d, 3000, lo=2, hi=9))
    win = tuple(int(rng.integers(1, s + 1)) for s in base_a.shape)
    sa = tuple(int(rng.integers(0, s - w + 1)) for s, w in zip(base_a.shape, win))
    base_b = rng.standard_normal(tuple(w + int(rng.integers(0, 3)) for w in win))
    sb = tuple(int(rng.integers(0, s - w + 1)) for s, w in zip(base_b.shape, win))
    base_c = np.full(tuple(w + 2 for w in win), 7.0)
    sc = (1,) * d
    ref = base_c.copy()
    O.apply_binary_view(ref, sc, base_a, sa, base_b, sb, win, "add")
    # describe the plan: dense shapes of the windows with base strides come from the view path,
    # so emulate it by offsetting flat buffers by each view's bias
    out = base_c.copy()
    bias = lambda st, bs: O.tuple_to_index(st, bs)
    desc = T.triot_plan_describe(1, [base_c.shape, base_a.shape, base_b.shape], win, d, F64, 0)
    # the dense plan of (base_c, base_a, base_b) over `win` has exactly the base strides; the
    # view plan adds the bias to each pointer, so run the model on the biased flat buffers
    kernel_model.run(desc, "binary", [out.reshape(-1)[bias(sc, base_c.shape):],
                                      base_a.reshape(-1)[bias(sa, base_a.shape):],
                                      base_b.reshape(-1)[bias(sb, base_b.shape):]], binop="add")
    np.testing.assert_array_equal(out, ref)


@pytest.mark.parametrize("seed", range(6))
def test_model_dot_and_update_vs_oracle(seed):
    rng = np.random.default_rng(5000 + seed)
    d = int(rng.integers(1, 7))
    ish = random_shape(rng, d, 2000, lo=1, hi=7 if d > 3 else 12)
    a = rng.integers(-50, 50, size=tuple(s + int(rng.integers(0, 3)) for s in ish)).astype(np.float64)
    b = rng.integers(-50, 50, size=tuple(s + int(rng.integers(0, 3)) for s in ish)).astype(np.float64)
    desc = T.triot_plan_describe(3, [a.shape, b.shape], ish, d, F64, 0, mode=seed % 2,
                                 warps=int(rng.integers(1, 6)))
    got = kernel_model.run(desc, "dot", [a.reshape(-1), b.reshape(-1)])
    assert got == O.inner_product(a, b, iter_shape=ish)          # integers: exact
    x = rng.standard_normal(ish)
    y = rng.standard_normal(tuple(s + int(rng.integers(0, 3)) for s in ish))
    z = rng.standard_normal(tuple(s + int(rng.integers(0, 3)) for s in ish))
    ref = x.copy()
    O.fused_update(ref, y, z)
    desc = T.triot_plan_describe(4, [x.shape, y.shape, z.shape], None, d, F64, 0,
                                 mode=seed % 2, warps=int(rng.integers(1, 6)))
    got = x.copy()
    kernel_model.run(desc, "update", [got.reshape(-1), y.reshape(-1), z.reshape(-1)])
    np.testing.assert_array_equal(_bits(got), _bits(ref))


def test_validation_dot_and_update():
    ws = T.triot_inner_product_workspace_size()
    st = T.triot_inner_product(FAKE, FAKE * 2, (3, 3), FAKE * 3, (3, 3), (4, 3), 2, F64, FAKE * 4,
                               ws, 0)
    assert st == 4
    # y smaller than x on an axis
    st = T.triot_fused_update(FAKE, (4, 4), FAKE * 2, (3, 4), FAKE * 3, (4, 4), 2, F64, 0)
    assert st == 4 and "'y'" in T.triot_last_error()
    st = T.triot_fused_update(FAKE, (4, 4), FAKE + 64, (4, 4), FAKE * 3, (4, 4), 2, F64, 0)
    assert st == 7


def test_validation_conv():
    st = T.triot_naive_convolve(FAKE, FAKE * 2, (3, 0), FAKE * 3, (2, 2), 2, F64, 0)
    assert st == 3
    st = T.triot_naive_convolve(FAKE * 2 + 8, FAKE * 2, (4, 4), FAKE * 3, (2, 2), 2, F64, 0)
    assert st == 7                                             # result overlaps lhs
    p = T.triot_plan_describe(5, [(256, 8), (256, 8)], None, 2, F64, 0)
    assert p["N"] == 511 * 15 and p["ext"] == [511, 15]


@pytest.fixture
def no_rows():
    """Row windows off for this thread (triot_set_launch_policy mode 5): embed and binary with
    short odd rows then take flat vectors."""
    lib = L.lib()
    assert lib.triot_set_launch_policy(5, 0) == 0
    yield
    lib.triot_set_launch_policy(-1, 0)


@pytest.mark.parametrize("seed", range(8))
def test_model_flat_vectors_vs_oracle(seed, no_rows):
    """Odd innermost extents take flat vectors (V consecutive counter elements across rows)."""
    _odd_shapes_vs_oracle(seed, expect="flat")


@pytest.mark.parametrize("seed", range(12))
def test_model_row_windows_vs_oracle(seed):
    """Short odd innermost extents take row windows for embed and binary (a lane per row, the
    warp sweeping the window's elements lane by lane); the expected value keeps flat vectors."""
    _odd_shapes_vs_oracle(seed, expect="rows")


def _odd_shapes_vs_oracle(seed, expect):
    rng = np.random.default_rng(6000 + seed)
    d = int(rng.integers(1, 6))
    odd = int(rng.choice([3, 5, 7, 9, 11]))
    dst_shape = random_shape(rng, d - 1, 800, lo=1, hi=9) + (odd,) if d > 1 else (odd * 37,)
    src_shape = tuple(max(1, s + int(rng.integers(-2, 2))) for s in dst_shape)
    dtype = "f32" if seed % 2 else "f64"
    dt = F32 if dtype == "f32" else F64
    src = random_values(rng, src_shape, dtype, "normal")
    ref = np.full(dst_shape, -7.0, dtype=src.dtype)
    O.embed(ref, src)
    region = seed % 3 == 2 and expect == "rows"
    if region:
        ref = np.full(dst_shape, -7.0, dtype=src.dtype)
        O.embed(ref, src, region_only=True)
    desc = T.triot_plan_describe(0, [dst_shape, src_shape], None, d, dt, 1 if region else 0,
                                 mode=seed % 2, warps=int(rng.integers(1, 6)))
    if not region or math.prod(min(a, b) for a, b in zip(dst_shape, src_shape)) > 1:
        assert desc[expect] or desc["V"] > 1 or desc["R"] > 1, desc
    out = np.full(dst_shape, -7.0, dtype=src.dtype)
    kernel_model.run(desc, "embed", [out.reshape(-1), src.reshape(-1)])
    np.testing.assert_array_equal(_bits(out), _bits(ref))
    # binary over the odd shape, c dense
    a = random_values(rng, tuple(s + int(rng.integers(0, 2)) for s in dst_shape), dtype, "normal")
    b = random_values(rng, dst_shape, dtype, "normal")
    refc = O.apply_binary(a, b, "mul", iter_shape=dst_shape)
    desc = T.triot_plan_describe(1, [None, a.shape, b.shape], dst_shape, d, dt, 2, mode=seed % 2,
                                 warps=int(rng.integers(1, 6)))
    c = np.full(dst_shape, 5.0, dtype=a.dtype)
    kernel_model.run(desc, "binary", [c.reshape(-1), a.reshape(-1), b.reshape(-1)], binop="mul")
    np.testing.assert_array_equal(_bits(c), _bits(refc))
    # expected value over the odd shape (integers: exact)
    p = rng.integers(0, 256, size=dst_shape).astype(np.float64)
    desc = T.triot_plan_describe(2, [dst_shape], None, d, F64, 0, mode=seed % 2,
                                 warps=int(rng.integers(1, 6)))
    got = kernel_model.run(desc, "ev", [p.reshape(-1)])
    np.testing.assert_array_equal(np.array(got), O.expected_value(p))


def test_ev_flat_64_byte_units_plan_and_model():
    """A dense expected value with an odd innermost extent longer than 64 bytes takes flat units
    of 64 bytes (at most one wrap per unit); shorter odd rows keep 32-byte flat vectors.  The CPU
    model of the flat walk (V elements with Alg 3's +1, then the mixed-radix skip) on that plan
    equals the oracle exactly on integer data."""
    p = T.triot_plan_describe(2, [(40, 33)], None, 2, F32, 0)
    assert p["flat"] and p["V"] == 16 and p["nvec"] == (40 * 33 + 15) // 16
    p = T.triot_plan_describe(2, [(40, 33)], None, 2, F64, 0)
    assert p["flat"] and p["V"] == 8
    p = T.triot_plan_describe(2, [(9, 17)], None, 2, F32, 0, [4, 0, 0])   # 17 > 16: 64-byte units
    assert p["flat"] and p["V"] == 16
    p = T.triot_plan_describe(2, [(9, 15)], None, 2, F32, 0, [4, 0, 0])   # short odd rows: 32 bytes
    assert p["flat"] and p["V"] == 8
    p = T.triot_plan_describe(2, [(9, 9)], None, 2, F64, 0, [8, 0, 0])    # 9 > 8: 64-byte units
    assert p["flat"] and p["V"] == 8
    rng = np.random.default_rng(64)
    for shape, dt, npdt in [((13, 33), F32, np.float32), ((7, 5, 19), F64, np.float64),
                            ((3, 4, 65), F32, np.float32), ((101,), F64, np.float64),
                            ((6, 9), F64, np.float64)]:
        q = rng.integers(0, 50, size=shape).astype(npdt)
        for warps in (1, 3, 8):
            desc = T.triot_plan_describe(2, [shape], None, len(shape), dt, 0, [8, 0, 0], 0, warps)
            assert desc["flat"] and desc["V"] * (4 if dt == F32 else 8) == 64
            got = kernel_model.run(desc, "ev", [q.reshape(-1)])
            np.testing.assert_array_equal(np.array(got), O.expected_value(q))


def test_ev_rows_that_would_take_16_byte_vectors():
    """A dense expected value whose rows only admit 16-byte vectors (12, 20, 28 floats; 6, 10, ...
    doubles) takes the shared-memory row tiles up to 31 elements and the 64-byte flat units beyond
    (32-byte aligned p), not half-width loads; views and rows of whole 32-byte vectors keep the
    regular geometry.  The CPU model on those plans equals the oracle."""
    for shape, dt in [((50, 12), F32), ((50, 20), F32), ((9, 7, 28), F32), ((50, 6), F64),
                      ((50, 10), F64), ((11, 30), F64)]:
        p = T.triot_plan_describe(2, [shape], None, len(shape), dt, 0)
        assert p["evrows"] and not p["flat"] and p["rowlen"] == shape[-1], (shape, p)
    for shape, dt, v in [((50, 36), F32, 16), ((50, 44), F32, 16), ((50, 34), F64, 8)]:
        p = T.triot_plan_describe(2, [shape], None, len(shape), dt, 0)
        assert p["flat"] and p["V"] == v, (shape, p)
        p = T.triot_plan_describe(2, [shape], None, len(shape), dt, 0, [16, 0, 0])
        assert not p["flat"] and not p["evrows"] and p["V"] * (4 if dt == F32 else 8) == 16
    p = T.triot_plan_describe(2, [(50, 16)], None, 2, F32, 0)
    assert not p["evrows"] and not p["flat"] and p["V"] == 8          # whole 32-byte vectors
    p = T.triot_plan_describe(2, [(50, 16)], None, 2, F32, 0, [16, 0, 0])
    assert p["evrows"]                              # 16-byte aligned only: rows of 16 as tiles
    rng = np.random.default_rng(16)
    for shape, dt, npdt in [((13, 12), F32, np.float32), ((5, 7, 6), F64, np.float64),
                            ((9, 36), F32, np.float32), ((3, 5, 34), F64, np.float64)]:
        q = rng.integers(0, 50, size=shape).astype(npdt)
        for warps in (1, 5):
            desc = T.triot_plan_describe(2, [shape], None, len(shape), dt, 0, [0, 0, 0], 0, warps)
            assert desc["evrows"] or desc["flat"]
            got = kernel_model.run(desc, "ev", [q.reshape(-1)])
            np.testing.assert_array_equal(np.array(got), O.expected_value(q))


def test_flat_geometry_chosen_for_odd_innermost(no_rows):
    p = T.triot_plan_describe(0, [(5, 7), (4, 6)], None, 2, F32, 0)
    assert p["flat"] and p["V"] == 8 and p["D"] == 2 and p["nvec"] == 5
    assert [t["vec"] for t in p["t"]] == [True, False]
    p = T.triot_plan_describe(2, [(7,) * 5], None, 5, F64, 0)
    assert p["flat"] and p["V"] == 4 and p["nvec"] == (7 ** 5 + 3) // 4
    p = T.triot_plan_describe(0, [(4, 8), (3, 8)], None, 2, F32, 0)
    assert not p["flat"]                       # a vector width fits: regular geometry


def test_row_window_geometry():
    """Short odd rows (<= 64) take row windows for embed / binary: the outer axes are the digits,
    one vector per row, dense tensors flagged; longer odd rows keep flat vectors."""
    p = T.triot_plan_describe(0, [(5, 7), (4, 6)], None, 2, F32, 0)
    assert p["rows"] and not p["flat"] and p["D"] == 1 and p["rowlen"] == 7
    assert (p["rmag"], p["nvec"], p["scols"], p["bnd"]) == ((1 << 32) // 7 + 1, 5, 6, [4])
    assert p["rwin"] == 3                                 # >= 16 elements per lane per group
    for n, w in ((3, 6), (5, 4), (9, 2), (15, 2), (17, 1), (63, 1)):
        q = T.triot_plan_describe(1, [None, (40, n), (39, n + 1)], (39, n), 2, F32, 2)
        assert q["rows"] and q["rwin"] == w and 32 * w * n + 32 * 8 <= (1 << 13), (n, q["rwin"])
    assert [t["vec"] for t in p["t"]] == [True, False]
    assert [t["tau"] for t in p["t"]] == [1, 1]
    p = T.triot_plan_describe(0, [(3000, 7), (2900, 5)], None, 2, F64, 0)
    assert p["rows"] and p["ext"] == [3000] and p["t"][1]["sig"] == [5]
    p = T.triot_plan_describe(0, [(11,), (4,)], None, 1, F32, 0)     # one row: a unit digit
    assert p["rows"] and p["D"] == 1 and p["ext"] == [1] and p["nvec"] == 1 and p["scols"] == 4
    p = T.triot_plan_describe(1, [None, (9, 65), (9, 66)], (9, 65), 2, F32, 2)
    assert p["flat"] and not p["rows"]                    # binary rows longer than 64: flat
    p = T.triot_plan_describe(0, [(9, 33), (8, 30)], None, 2, F32, 0)
    assert p["flat"] and not p["rows"]                    # embed rows longer than 31: flat
    p = T.triot_plan_describe(0, [(9, 31), (8, 30)], None, 2, F32, 0)
    assert p["rows"]
    p = T.triot_plan_describe(1, [None, (9, 63), (9, 66)], (9, 63), 2, F32, 2)
    assert p["rows"] and [t["vec"] for t in p["t"]] == [True, True, False]
    p = T.triot_plan_describe(2, [(7,) * 5], None, 5, F64, 0)
    # the dense expected value of short odd rows: shared-memory row tiles over the outer digits
    assert p["evrows"] and not p["flat"] and not p["rows"] and p["D"] == 4 and p["rowlen"] == 7
    assert p["nvec"] == 7 ** 4 and p["slot_of_axis"] == [0, 1, 2, 3, 4, 5]
    # ... unless p is not 16-byte aligned (the bulk copies) or the row is too long: flat vectors
    p = T.triot_plan_describe(2, [(7,) * 5], None, 5, F64, 0, [8, 0, 0])
    assert p["flat"] and not p["evrows"]
    p = T.triot_plan_describe(2, [(40, 33)], None, 2, F32, 0)
    assert p["flat"] and not p["evrows"]


def test_row_window_division_magic_exact():
    """umulhi(e, 2^32 // n + 1) == e // n for every row length the row windows take (3..64) and
    every element index a group of windows (plus a batch of overrun) can reach."""
    e = np.arange(1 << 13, dtype=np.uint64)
    for n in range(3, 65):
        mg = (1 << 32) // n + 1
        assert mg < (1 << 32)
        assert np.array_equal((e * np.uint64(mg)) >> np.uint64(32), e // np.uint64(n)), n
    # long rows (misaligned outputs): one window per group, e < 32 n + 256, up to n = 4096
    for n in list(range(249, 300)) + [383, 384, 511, 512, 999, 1000, 2047, 3001, 4095, 4096]:
        e = np.arange(32 * n + 256, dtype=np.uint64)
        mg = (1 << 32) // n + 1
        assert np.array_equal((e * np.uint64(mg)) >> np.uint64(32), e // np.uint64(n)), n


def test_row_windows_for_misaligned_outputs():
    """An output whose base is only element-aligned takes row windows (rows <= 4096) instead of
    element stores at a 32-byte lane stride; an aligned one keeps 32-byte vectors."""
    p = T.triot_plan_describe(0, [(512,) * 3, (384,) * 3], None, 3, F32, 0, ptr_mod32=(4, 0, 0))
    assert p["dshift"] == 1 and not p["rows"]            # embed, dense dst: shifted 32-B stores
    p = T.triot_plan_describe(0, [(512,) * 3, (384,) * 3], None, 3, F32, 0)
    assert not p["rows"] and p["V"] == 8 and p["dshift"] == 0
    p = T.triot_plan_describe(1, [(512,) * 3, (512,) * 3, (520,) * 3], (512,) * 3, 3, F32, 2,
                              ptr_mod32=(4, 0, 0))
    assert p["dshift"] == 1 and not p["rows"]            # binary, dense c: shifted stores
    p = T.triot_plan_describe(1, [(64, 100), (64, 100), (64, 96)], (64, 96), 2, F64, 2,
                              ptr_mod32=(8, 0, 0))
    assert p["rows"] and p["rowlen"] == 96               # c wider than the iteration: rows
    p = T.triot_plan_describe(0, [(4, 8192), (4, 8000)], None, 2, F32, 1, ptr_mod32=(4, 0, 0))
    assert p["rows"] and (p["seglen"], p["segm"], p["rowlen"]) == (500, 8000, 500)  # segments
    p = T.triot_plan_describe(1, [(4, 8191), (4, 8191), (4, 8191)], None, 2, F32, 2,
                              ptr_mod32=(4, 0, 0))
    assert not p["rows"]                 # merged 4 x 8191 (prime): no segment length in [64, 512]


@pytest.mark.parametrize("seed", range(10))
def test_model_misaligned_output_rows_vs_oracle(seed):
    """Row windows planned for misaligned outputs (long rows, one window per group) run through
    the kernel model bit-exact against the oracle."""
    rng = np.random.default_rng(8000 + seed)
    d = int(rng.integers(1, 4))
    n = int(rng.choice([8, 16, 40, 45, 256, 300, 383]))
    dst_shape = random_shape(rng, d - 1, 4000 // n + 2, lo=1, hi=12) + (n,) if d > 1 else (n,)
    src_shape = tuple(max(1, s + int(rng.integers(-2, 3))) for s in dst_shape)
    src = random_values(rng, src_shape, "f32", "normal")
    region = seed % 2 == 1
    ref = np.full(dst_shape, -7.0, dtype=np.float32)
    O.embed(ref, src, region_only=region)
    desc = T.triot_plan_describe(0, [dst_shape, src_shape], None, d, F32, 1 if region else 0,
                                 ptr_mod32=(4, 0, 0), mode=0, warps=int(rng.integers(1, 6)))
    assert desc["rows"] or desc["dshift"] or desc["V"] == 1, desc
    out = np.full(dst_shape, -7.0, dtype=np.float32)
    kernel_model.run(desc, "embed", [out.reshape(-1), src.reshape(-1)])
    np.testing.assert_array_equal(_bits(out), _bits(ref))


def test_row_windows_for_odd_rows_into_non_dense_outputs():
    """Odd rows longer than the dense thresholds still take row windows when the output is not
    dense in the counter (region-only embed, a c larger than the iteration) or misaligned."""
    p = T.triot_plan_describe(0, [(40, 383), (40, 383)], None, 2, F32, 0, ptr_mod32=(4, 0, 0))
    assert p["dshift"] == 1 and p["V"] == 8                # merged 15320, dense dst: shifted
    p = T.triot_plan_describe(0, [(40, 383), (30, 380)], None, 2, F32, 0)
    assert p["flat"]                                       # dense aligned dst: flat vectors
    p = T.triot_plan_describe(0, [(40, 383), (30, 380)], None, 2, F32, 0, ptr_mod32=(4, 0, 0))
    assert p["rows"]                                       # misaligned dst: row windows
    p = T.triot_plan_describe(0, [(40, 383), (30, 380)], None, 2, F32, 1)
    assert p["rows"] and not p["t"][0]["vec"]              # region only: dst rows of 383 > 380
    p = T.triot_plan_describe(1, [(40, 200), (40, 99), (40, 99)], (40, 99), 2, F64, 2)
    assert p["rows"] and not p["t"][0]["vec"]              # c wider than the iteration


def test_pow2_decode_and_linear_tensor0_flags():
    """The plan flags shift decoding when every digit extent is a power of two, and the linear
    offset of a tensor 0 dense in the digit space (C2, C3, C5 yes; C4's 24 is not a power of
    two; a wide c is not dense)."""
    c5 = T.triot_plan_describe(0, [(4,) * 14, (3,) * 14], None, 14, F32, 0)
    assert c5["pow2"] and c5["lin0"] == 8
    c2 = T.triot_plan_describe(0, [(512,) * 3, (384,) * 3], None, 3, F32, 0)
    assert c2["pow2"] and c2["lin0"] == 8
    c4 = T.triot_plan_describe(1, [None, (32, 48, 24, 40, 36), (40, 32, 32, 32, 32)],
                               (32, 32, 24, 32, 32), 5, F64, 2)
    assert not c4["pow2"] and c4["lin0"] == 4
    wide = T.triot_plan_describe(1, [(8, 40), (8, 32), (8, 32)], (8, 32), 2, F64, 2)
    assert wide["lin0"] == 0
    ev = T.triot_plan_describe(2, [(16,) * 6], None, 6, F64, 0)
    assert ev["pow2"]


@pytest.mark.parametrize("seed", range(8))
def test_model_segmented_rows_vs_oracle(seed):
    """Fully merged long rows into a misaligned output are cut into segments (rows of a divisor
    L <= 4096 of the merged extent, per-segment embed bound): the kernel model is bit-exact
    against the oracle for pads, crops and binary ops."""
    rng = np.random.default_rng(9000 + seed)
    n1 = int(rng.choice([2, 3, 5]))
    inner = int(rng.choice([1024, 1500, 2048, 3000]))
    dst_shape = (int(rng.integers(3, 7)), n1, inner)
    src_shape = (dst_shape[0] + int(rng.integers(-2, 2)), n1, inner)   # inner axes merge
    src = random_values(rng, src_shape, "f32", "normal")
    ref = np.full(dst_shape, -7.0, dtype=np.float32)
    O.embed(ref, src)
    desc = T.triot_plan_describe(0, [dst_shape, src_shape], None, 3, F32, 0,
                                 ptr_mod32=(4, 0, 0), mode=0, warps=int(rng.integers(1, 5)))
    assert desc["dshift"] == 1, desc                        # embed: shifted 32-B stores
    out = np.full(dst_shape, -7.0, dtype=np.float32)
    kernel_model.run(desc, "embed", [out.reshape(-1), src.reshape(-1)])
    np.testing.assert_array_equal(_bits(out), _bits(ref))
    a = random_values(rng, dst_shape, "f32", "normal")
    b = random_values(rng, dst_shape, "f32", "normal")
    cs = dst_shape[:-1] + (dst_shape[-1] + 8,)            # c wider: not dense, rows > 512
    refc = np.full(cs, 5.0, dtype=np.float32)
    O.apply_binary(a, b, "add", out=refc)
    desc = T.triot_plan_describe(1, [cs, dst_shape, dst_shape], dst_shape, 3, F32, 0,
                                 ptr_mod32=(4, 0, 0), mode=0, warps=int(rng.integers(1, 5)))
    assert desc["rows"] and desc["seglen"] > 0, desc
    c = np.full(cs, 5.0, dtype=np.float32)
    kernel_model.run(desc, "binary", [c.reshape(-1), a.reshape(-1), b.reshape(-1)], binop="add")
    np.testing.assert_array_equal(_bits(c), _bits(refc))


def test_warp_per_row_plan_rule():
    """Long rows (>= 128) into an output not dense in the counter take a warp per row; dense
    outputs and short rows keep the row table."""
    p = T.triot_plan_describe(1, [(512,) * 3, (512,) * 3, (520,) * 3], (512,) * 3, 3, F32, 2,
                              ptr_mod32=(4, 0, 0))
    assert p["dshift"] == 1 and not p["rows"]             # dense misaligned c: shifted stores
    p = T.triot_plan_describe(0, [(41, 400), (40, 383)], None, 2, F32, 1)
    assert p["rows"] and p["rwarp"]                       # region only, rows of 383
    p = T.triot_plan_describe(1, [(40, 200), (40, 99), (40, 99)], (40, 99), 2, F64, 2)
    assert p["rows"] and not p["rwarp"]                   # rows of 99 < 128: table
    p = T.triot_plan_describe(1, [(40, 300), (40, 199), (40, 199)], (40, 199), 2, F64, 2)
    assert p["rows"] and p["rwarp"]                       # wide c, rows of 199


def test_shifted_store_plan():
    """An embed whose dst is dense in the counter but misaligned by whole elements keeps 32-B
    vectors and stores them shifted (dshift = misalignment in elements); aligned, view and
    region-only destinations do not."""
    for esz, dt in ((4, F32), (8, F64)):
        for k in range(1, 32 // esz):
            p = T.triot_plan_describe(0, [(64, 64), (60, 60)], None, 2, dt, 0,
                                      ptr_mod32=(k * esz, 0, 0))
            assert p["dshift"] == k and p["V"] == 32 // esz, (esz, k, p["dshift"])
    assert T.triot_plan_describe(0, [(64, 64), (60, 60)], None, 2, F32, 0)["dshift"] == 0
    p = T.triot_plan_describe(0, [(64, 64), (60, 60)], None, 2, F32, 1, ptr_mod32=(4, 0, 0))
    assert p["dshift"] == 0                               # region only: dst rows not dense



@pytest.mark.parametrize("seed", range(4))
def test_planner_never_selects_uncompiled_instances(seed):
    """inst.cu compiles no one-element-vector instances for embed, binary and the dense expected
    value, and no zero-run instance for D = 1: over random shapes, alignments and policies the
    planner never selects them (a V = 1 plan is always flat vectors or row windows)."""
    rng = np.random.default_rng(900 + seed)
    for trial in range(300):
        d = int(rng.integers(1, 9))
        dt = [F32, F64][trial % 2]
        a = random_shape(rng, d, 4000, lo=1, hi=9)
        b = tuple(int(x) + int(rng.integers(0, 3)) for x in a)
        mods = [int(rng.integers(0, 8)) * (4 if dt == F32 else 8) % 32 for _ in range(3)]
        plans = [T.triot_plan_describe(0, [b, a], None, d, dt, 0, mods),
                 T.triot_plan_describe(0, [a, b], None, d, dt, 0, mods),
                 T.triot_plan_describe(1, [None, a, b], None, d, dt, 2, mods),
                 T.triot_plan_describe(1, [b, a, b], a, d, dt, 0, mods),
                 T.triot_plan_describe(2, [a], None, d, dt, 0, mods)]
        for pl in plans:
            if pl["empty"]:
                continue
            assert pl["V"] > 1 or pl["flat"] or pl["rows"] or pl["evrows"], pl
            assert not (pl["zmask"] and pl["D"] < 2), pl
