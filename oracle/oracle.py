"""ctypes front end of the CPU oracle (oracle/triot_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs, never by the product package.  It builds
liboracle.so with gcc on first use (-O2 -fno-fast-math -ffp-contract=off, single thread)
and exposes the paper's definitions on numpy arrays.  See the C file's header for the
paper passage each function follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "triot_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_CFLAGS = ["-O2", "-fno-fast-math", "-ffp-contract=off", "-fPIC", "-shared", "-std=c11"]
_lock = threading.Lock()
_lib = None

F32, F64 = 0, 1
ADD, SUB, MUL, DIV = 0, 1, 2, 3
OPS = {"add": ADD, "sub": SUB, "mul": MUL, "div": DIV}

_u64p = ctypes.POINTER(ctypes.c_uint64)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_dblp = ctypes.POINTER(ctypes.c_double)


def build(force: bool = False) -> str:
    """Compile liboracle.so if it is missing or older than the C source."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.run(["gcc", *_CFLAGS, "-o", tmp, _SRC], check=True)
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            L.oracle_tuple_to_index.restype = ctypes.c_uint64
            L.oracle_tuple_to_index.argtypes = [_u64p, _u64p, ctypes.c_uint]
            L.oracle_advance_tuple.restype = None
            L.oracle_advance_tuple.argtypes = [_u64p, _u64p, ctypes.c_uint]
            L.oracle_index_to_tuple.restype = None
            L.oracle_index_to_tuple.argtypes = [ctypes.c_uint64, _u64p, ctypes.c_uint, _u64p]
            L.oracle_reindex.restype = ctypes.c_uint64
            L.oracle_reindex.argtypes = [ctypes.c_uint64, _u64p, _u64p, ctypes.c_uint]
            L.oracle_reindex_powers_of_2.restype = ctypes.c_uint64
            L.oracle_reindex_powers_of_2.argtypes = [ctypes.c_uint64, _u32p, _u32p, ctypes.c_uint]
            L.oracle_enumerate.restype = None
            L.oracle_enumerate.argtypes = [_u64p, ctypes.c_uint, _u64p]
            L.oracle_embed.restype = None
            L.oracle_embed.argtypes = [ctypes.c_void_p, _u64p, ctypes.c_void_p, _u64p,
                                       ctypes.c_uint, ctypes.c_uint, ctypes.c_int]
            L.oracle_apply_binary.restype = None
            L.oracle_apply_binary.argtypes = [ctypes.c_void_p, _u64p, ctypes.c_void_p, _u64p,
                                              ctypes.c_void_p, _u64p, _u64p, ctypes.c_uint,
                                              ctypes.c_int, ctypes.c_int]
            L.oracle_expected_value.restype = None
            L.oracle_expected_value.argtypes = [_dblp, _dblp, ctypes.c_void_p, _u64p,
                                                ctypes.c_uint, ctypes.c_int]
            L.oracle_expected_value_abs.restype = None
            L.oracle_expected_value_abs.argtypes = [_dblp, ctypes.c_void_p, _u64p,
                                                    ctypes.c_uint, ctypes.c_int]
            L.oracle_view_bias.restype = ctypes.c_uint64
            L.oracle_view_bias.argtypes = [_u64p, _u64p, ctypes.c_uint]
            L.oracle_embed_view.restype = None
            L.oracle_embed_view.argtypes = [ctypes.c_void_p, _u64p, _u64p, _u64p,
                                            ctypes.c_void_p, _u64p, _u64p, _u64p,
                                            ctypes.c_uint, ctypes.c_uint, ctypes.c_int]
            L.oracle_apply_binary_view.restype = None
            L.oracle_apply_binary_view.argtypes = [ctypes.c_void_p, _u64p, _u64p,
                                                   ctypes.c_void_p, _u64p, _u64p,
                                                   ctypes.c_void_p, _u64p, _u64p, _u64p,
                                                   ctypes.c_uint, ctypes.c_int, ctypes.c_int]
            L.oracle_inner_product.restype = None
            L.oracle_inner_product.argtypes = [_dblp, _dblp, ctypes.c_void_p, _u64p,
                                               ctypes.c_void_p, _u64p, _u64p, ctypes.c_uint,
                                               ctypes.c_int]
            L.oracle_fused_update.restype = None
            L.oracle_fused_update.argtypes = [ctypes.c_void_p, _u64p, ctypes.c_void_p, _u64p,
                                              ctypes.c_void_p, _u64p, ctypes.c_uint,
                                              ctypes.c_int]
            L.oracle_naive_convolve.restype = None
            L.oracle_naive_convolve.argtypes = [ctypes.c_void_p, ctypes.c_void_p, _u64p,
                                                ctypes.c_void_p, _u64p, ctypes.c_uint,
                                                ctypes.c_int]
            _lib = L
    return _lib


def _shape(s) -> ctypes.Array:
    return (ctypes.c_uint64 * max(1, len(s)))(*[int(x) for x in s])


def _dtype_code(arr: np.ndarray) -> int:
    if arr.dtype == np.float32:
        return F32
    if arr.dtype == np.float64:
        return F64
    raise TypeError("oracle supports float32 and float64, got %s" % arr.dtype)


def _ptr(arr: np.ndarray) -> int:
    assert arr.flags["C_CONTIGUOUS"]
    return arr.ctypes.data


# -- L0 ---------------------------------------------------------------------------------------

def tuple_to_index(tup, shape) -> int:
    """Alg 2."""
    return int(lib().oracle_tuple_to_index(_shape(tup), _shape(shape), len(shape)))


def advance_tuple(tup, shape) -> tuple:
    """Alg 3; returns the advanced tuple."""
    t = _shape(tup)
    lib().oracle_advance_tuple(t, _shape(shape), len(shape))
    return tuple(int(x) for x in t[: len(shape)])


def index_to_tuple(index: int, shape) -> tuple:
    """P:139 derivation (% then /)."""
    out = (ctypes.c_uint64 * len(shape))()
    lib().oracle_index_to_tuple(int(index), _shape(shape), len(shape), out)
    return tuple(int(x) for x in out)


def reindex(index: int, shape, new_shape) -> int:
    """Alg 4."""
    return int(lib().oracle_reindex(int(index), _shape(shape), _shape(new_shape), len(shape)))


def reindex_powers_of_2(index: int, log_shape, new_log_shape) -> int:
    """Alg 12."""
    a = (ctypes.c_uint32 * len(log_shape))(*log_shape)
    b = (ctypes.c_uint32 * len(new_log_shape))(*new_log_shape)
    return int(lib().oracle_reindex_powers_of_2(int(index), a, b, len(log_shape)))


def enumerate_tuples(shape) -> np.ndarray:
    """All tuples of shape in Alg 3 order, as an (N, d) uint64 array."""
    n = int(np.prod(shape, dtype=np.uint64)) if len(shape) else 0
    out = np.zeros((n, len(shape)), dtype=np.uint64)
    if n:
        lib().oracle_enumerate(_shape(shape), len(shape),
                               out.ctypes.data_as(_u64p))
    return out


# -- L4: the three operations -------------------------------------------------------------------

def embed(dst: np.ndarray, src: np.ndarray, region_only: bool = False) -> np.ndarray:
    """In place on dst; returns dst."""
    assert dst.dtype == src.dtype and dst.ndim == src.ndim
    lib().oracle_embed(_ptr(dst), _shape(dst.shape), _ptr(src), _shape(src.shape),
                       dst.ndim, dst.itemsize, 1 if region_only else 0)
    return dst


def apply_binary(a: np.ndarray, b: np.ndarray, op: str = "mul", iter_shape=None,
                 out: np.ndarray | None = None) -> np.ndarray:
    """c[t] = a[t] OP b[t] for t in iter_shape (default elementwise min)."""
    assert a.dtype == b.dtype and a.ndim == b.ndim
    if iter_shape is None:
        iter_shape = tuple(min(x, y) for x, y in zip(a.shape, b.shape))
    if out is None:
        out = np.empty(iter_shape, dtype=a.dtype)
    lib().oracle_apply_binary(_ptr(out), _shape(out.shape), _ptr(a), _shape(a.shape),
                              _ptr(b), _shape(b.shape), _shape(iter_shape), a.ndim,
                              _dtype_code(a), OPS[op])
    return out


def expected_value(p: np.ndarray, with_plain: bool = False):
    """Alg 11: m_k = sum_t t_k p[t], fp64, Neumaier-compensated."""
    d = p.ndim
    means = (ctypes.c_double * d)()
    plain = (ctypes.c_double * d)()
    lib().oracle_expected_value(means, plain, _ptr(p), _shape(p.shape), d, _dtype_code(p))
    m = np.array(means[:d], dtype=np.float64)
    if with_plain:
        return m, np.array(plain[:d], dtype=np.float64)
    return m


def expected_value_abs(p: np.ndarray) -> np.ndarray:
    """sum_t |t_k p[t]| per axis (the scale of the relative bound for signed inputs)."""
    d = p.ndim
    out = (ctypes.c_double * d)()
    lib().oracle_expected_value_abs(out, _ptr(p), _shape(p.shape), d, _dtype_code(p))
    return np.array(out[:d], dtype=np.float64)


# -- NEXT-1: views ------------------------------------------------------------

def view_bias(start, base_shape) -> int:
    """bias = tuple_to_index(start, base_shape)."""
    return int(lib().oracle_view_bias(_shape(start), _shape(base_shape), len(base_shape)))


def embed_view(dst_base: np.ndarray, dst_start, dst_window, src_base: np.ndarray, src_start,
               src_window, region_only: bool = False) -> np.ndarray:
    """In place on dst_base: the dst window receives the zero-padded src window."""
    assert dst_base.dtype == src_base.dtype and dst_base.ndim == src_base.ndim
    d = dst_base.ndim
    lib().oracle_embed_view(_ptr(dst_base), _shape(dst_base.shape), _shape(dst_start),
                            _shape(dst_window), _ptr(src_base), _shape(src_base.shape),
                            _shape(src_start), _shape(src_window), d, dst_base.itemsize,
                            1 if region_only else 0)
    return dst_base


def apply_binary_view(c_base: np.ndarray, c_start, a_base: np.ndarray, a_start,
                      b_base: np.ndarray, b_start, iter_shape, op: str = "mul") -> np.ndarray:
    """In place on c_base: c_view[t] = a_view[t] OP b_view[t] for t in iter_shape."""
    d = a_base.ndim
    lib().oracle_apply_binary_view(_ptr(c_base), _shape(c_base.shape), _shape(c_start),
                                   _ptr(a_base), _shape(a_base.shape), _shape(a_start),
                                   _ptr(b_base), _shape(b_base.shape), _shape(b_start),
                                   _shape(iter_shape), d, _dtype_code(a_base), OPS[op])
    return c_base


# -- NEXT-2 / NEXT-3: Benchmarks 2 and 3 --------------------------------------------------

def inner_product(a: np.ndarray, b: np.ndarray, iter_shape=None, with_plain: bool = False):
    """Alg 8 dot_product over iter_shape (default: the shared tuples, min shape)."""
    assert a.dtype == b.dtype and a.ndim == b.ndim
    if iter_shape is None:
        iter_shape = tuple(min(x, y) for x, y in zip(a.shape, b.shape))
    out, plain = ctypes.c_double(0.0), ctypes.c_double(0.0)
    lib().oracle_inner_product(ctypes.byref(out), ctypes.byref(plain), _ptr(a), _shape(a.shape),
                               _ptr(b), _shape(b.shape), _shape(iter_shape), a.ndim,
                               _dtype_code(a))
    return (out.value, plain.value) if with_plain else out.value


def fused_update(x: np.ndarray, y: np.ndarray, z: np.ndarray) -> np.ndarray:
    """Benchmark 3, in place on x: x[t] = x[t] + y[t]*x[t] - z[t] over x's shape."""
    assert x.dtype == y.dtype == z.dtype and x.ndim == y.ndim == z.ndim
    lib().oracle_fused_update(_ptr(x), _shape(x.shape), _ptr(y), _shape(y.shape), _ptr(z),
                              _shape(z.shape), x.ndim, _dtype_code(x))
    return x


# -- NEXT-4: naive convolution, Alg 15 ---------------------------------------------

def naive_convolve(lhs: np.ndarray, rhs: np.ndarray) -> np.ndarray:
    """Alg 15: result (shape lhs + rhs - 1) with result[t_l + t_r] += lhs[t_l] * rhs[t_r]."""
    assert lhs.dtype == rhs.dtype and lhs.ndim == rhs.ndim
    out = np.empty(tuple(a + b - 1 for a, b in zip(lhs.shape, rhs.shape)), dtype=lhs.dtype)
    lib().oracle_naive_convolve(_ptr(out), _ptr(lhs), _shape(lhs.shape), _ptr(rhs),
                                _shape(rhs.shape), lhs.ndim, _dtype_code(lhs))
    return out
