"""ctypes binding of libtriot.so -- argument marshalling only.

The functions here have the C-ABI's names and arguments (include/triot.h): raw device
pointers as ints, shapes as sequences of ints, the CUDA stream as an int handle.  Every step
of the hot path runs in the library's sm_100a kernels; there is no Python or CPU fallback:
if the library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes
import json
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# TRIOT_LIB_PATH: an alternative build of the same library (A/B measurements in tools/ only)
LIB_PATH = os.environ.get("TRIOT_LIB_PATH") or os.path.join(_PKG, "libtriot.so")

TRIOT_F32, TRIOT_F64 = 0, 1
TRIOT_ADD, TRIOT_SUB, TRIOT_MUL, TRIOT_DIV = 0, 1, 2, 3
TRIOT_EMBED_FULL, TRIOT_EMBED_REGION_ONLY = 0, 1
OP_EMBED, OP_BINARY, OP_EV, OP_DOT, OP_UPDATE, OP_CONV = 0, 1, 2, 3, 4, 5

STATUS = {
    0: "TRIOT_OK", 1: "TRIOT_ERR_NULL_POINTER", 2: "TRIOT_ERR_UNSUPPORTED_DIMENSION",
    3: "TRIOT_ERR_BAD_SHAPE", 4: "TRIOT_ERR_AXIS_OUT_OF_BOUNDS", 5: "TRIOT_ERR_BAD_DTYPE_OR_OP",
    6: "TRIOT_ERR_MISALIGNED", 7: "TRIOT_ERR_ALIASING", 8: "TRIOT_ERR_WORKSPACE",
    9: "TRIOT_ERR_CUDA",
}
EXPORTS = ("triot_max_dimension", "triot_status_string", "triot_last_error", "triot_embed",
           "triot_apply_binary", "triot_expected_value_workspace_size", "triot_expected_value",
           "triot_expected_value_mass", "triot_embed_view", "triot_apply_binary_view",
           "triot_expected_value_view",
           "triot_inner_product_workspace_size", "triot_inner_product", "triot_fused_update",
           "triot_naive_convolve", "triot_embed_host", "triot_apply_binary_host",
           "triot_plan_describe", "triot_set_launch_policy", "triot_fastdiv_magic",
           "triot_expected_value_offset", "triot_sum_rows", "triot_expected_value_host")


class TriotError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS.get(status, status)}: {message}")
        self.status = status
        self.message = message


if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python paper_1608_00099_b200/build.py` "
        "(there is no CPU fallback)")

_lib = ctypes.CDLL(LIB_PATH)
_i64p = ctypes.POINTER(ctypes.c_int64)
_vp = ctypes.c_void_p

_lib.triot_max_dimension.restype = ctypes.c_int
_lib.triot_max_dimension.argtypes = []
_lib.triot_status_string.restype = ctypes.c_char_p
_lib.triot_status_string.argtypes = [ctypes.c_int]
_lib.triot_last_error.restype = ctypes.c_char_p
_lib.triot_last_error.argtypes = []
_lib.triot_embed.restype = ctypes.c_int
_lib.triot_embed.argtypes = [_vp, _i64p, _vp, _i64p, ctypes.c_int, ctypes.c_int, ctypes.c_uint,
                             _vp]
_lib.triot_apply_binary.restype = ctypes.c_int
_lib.triot_apply_binary.argtypes = [_vp, _i64p, _vp, _i64p, _vp, _i64p, _i64p, ctypes.c_int,
                                    ctypes.c_int, ctypes.c_int, _vp]
_lib.triot_expected_value_workspace_size.restype = ctypes.c_int
_lib.triot_expected_value_workspace_size.argtypes = [_i64p, ctypes.c_int, ctypes.c_int,
                                                     ctypes.POINTER(ctypes.c_size_t)]
_lib.triot_expected_value.restype = ctypes.c_int
_lib.triot_expected_value.argtypes = [_vp, _vp, _i64p, ctypes.c_int, ctypes.c_int, _vp,
                                      ctypes.c_size_t, _vp]
_lib.triot_expected_value_mass.restype = ctypes.c_int
_lib.triot_expected_value_mass.argtypes = _lib.triot_expected_value.argtypes
_lib.triot_expected_value_offset.restype = ctypes.c_int
_lib.triot_expected_value_offset.argtypes = [ctypes.c_void_p, ctypes.c_void_p, _i64p, _i64p,
                                             ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                             ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
_lib.triot_sum_rows.restype = ctypes.c_int
_lib.triot_sum_rows.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                ctypes.c_void_p]
_lib.triot_expected_value_host.restype = ctypes.c_int
_lib.triot_expected_value_host.argtypes = [ctypes.c_void_p, ctypes.c_void_p, _i64p, _i64p,
                                           ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
class triot_view(ctypes.Structure):
    """include/triot.h triot_view: a window of a dense base tensor."""
    _fields_ = [("data", ctypes.c_void_p), ("base_shape", _i64p), ("start", _i64p),
                ("shape", _i64p)]


_viewp = ctypes.POINTER(triot_view)
_lib.triot_embed_view.restype = ctypes.c_int
_lib.triot_embed_view.argtypes = [_viewp, _viewp, ctypes.c_int, ctypes.c_int, ctypes.c_uint, _vp]
_lib.triot_apply_binary_view.restype = ctypes.c_int
_lib.triot_apply_binary_view.argtypes = [_viewp, _viewp, _viewp, _i64p, ctypes.c_int,
                                         ctypes.c_int, ctypes.c_int, _vp]
_lib.triot_expected_value_view.restype = ctypes.c_int
_lib.triot_expected_value_view.argtypes = [_vp, _viewp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                           _vp, ctypes.c_size_t, _vp]
_lib.triot_inner_product_workspace_size.restype = ctypes.c_int
_lib.triot_inner_product_workspace_size.argtypes = [ctypes.POINTER(ctypes.c_size_t)]
_lib.triot_inner_product.restype = ctypes.c_int
_lib.triot_inner_product.argtypes = [_vp, _vp, _i64p, _vp, _i64p, _i64p, ctypes.c_int,
                                     ctypes.c_int, _vp, ctypes.c_size_t, _vp]
_lib.triot_fused_update.restype = ctypes.c_int
_lib.triot_fused_update.argtypes = [_vp, _i64p, _vp, _i64p, _vp, _i64p, ctypes.c_int,
                                    ctypes.c_int, _vp]
_lib.triot_naive_convolve.restype = ctypes.c_int
_lib.triot_naive_convolve.argtypes = [_vp, _vp, _i64p, _vp, _i64p, ctypes.c_int, ctypes.c_int,
                                      _vp]
_lib.triot_embed_host.restype = ctypes.c_int
_lib.triot_embed_host.argtypes = [_vp, _i64p, _vp, _i64p, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_uint, _vp, ctypes.c_size_t, _vp]
_lib.triot_apply_binary_host.restype = ctypes.c_int
_lib.triot_apply_binary_host.argtypes = [_vp, _vp, _i64p, _vp, _i64p, _i64p, ctypes.c_int,
                                         ctypes.c_int, ctypes.c_int, _vp, ctypes.c_size_t, _vp]
_lib.triot_plan_describe.restype = ctypes.c_int
_lib.triot_plan_describe.argtypes = [ctypes.c_int, ctypes.POINTER(_i64p), _i64p, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_uint, ctypes.POINTER(ctypes.c_uint),
                                     ctypes.c_int, ctypes.c_uint64, ctypes.c_char_p,
                                     ctypes.c_size_t]
_lib.triot_set_launch_policy.restype = ctypes.c_int
_lib.triot_set_launch_policy.argtypes = [ctypes.c_int, ctypes.c_int]
_lib.triot_fastdiv_magic.restype = ctypes.c_int
_lib.triot_fastdiv_magic.argtypes = [ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint32),
                                     ctypes.POINTER(ctypes.c_uint32)]


def lib() -> ctypes.CDLL:
    return _lib


_SHAPES: dict = {}   # shape tuple -> its int64_t[] (the C side only reads it): ~2 us per call saved


def _shape(s):
    if s is None:
        return None
    try:
        return _SHAPES[s]
    except (KeyError, TypeError):
        pass
    t = tuple(int(x) for x in s)
    arr = (ctypes.c_int64 * max(1, len(t)))(*t)
    if len(_SHAPES) < 4096 and not isinstance(s, list):
        _SHAPES[t] = arr
    return arr


def check(status: int) -> None:
    if status != 0:
        raise TriotError(status, _lib.triot_last_error().decode())


# ---- the C-ABI, one Python function per entry point (same names) --------------------------

def triot_max_dimension() -> int:
    return _lib.triot_max_dimension()


def triot_status_string(status: int) -> str:
    return _lib.triot_status_string(status).decode()


def triot_last_error() -> str:
    return _lib.triot_last_error().decode()


def triot_embed(dst: int, dst_shape, src: int, src_shape, d: int, dtype: int, flags: int,
                stream: int) -> int:
    return _lib.triot_embed(dst, _shape(dst_shape), src, _shape(src_shape), d, dtype, flags,
                            stream)


def triot_apply_binary(c: int, c_shape, a: int, a_shape, b: int, b_shape, iter_shape, d: int,
                       dtype: int, op: int, stream: int) -> int:
    return _lib.triot_apply_binary(c, _shape(c_shape), a, _shape(a_shape), b, _shape(b_shape),
                                   _shape(iter_shape), d, dtype, op, stream)


def triot_expected_value_workspace_size(shape, d: int, dtype: int) -> int:
    out = ctypes.c_size_t(0)
    check(_lib.triot_expected_value_workspace_size(_shape(shape), d, dtype, ctypes.byref(out)))
    return int(out.value)


def triot_expected_value(means: int, p: int, shape, d: int, dtype: int, workspace: int,
                         workspace_bytes: int, stream: int) -> int:
    return _lib.triot_expected_value(means, p, _shape(shape), d, dtype, workspace,
                                     workspace_bytes, stream)


def triot_expected_value_mass(out: int, p: int, shape, d: int, dtype: int, workspace: int,
                              workspace_bytes: int, stream: int) -> int:
    return _lib.triot_expected_value_mass(out, p, _shape(shape), d, dtype, workspace,
                                          workspace_bytes, stream)


def make_view(data: int, base_shape, start, shape):
    """A triot_view plus the arrays it points to (keep the tuple alive during the call)."""
    bs, st, sh = _shape(base_shape), _shape(start) if start is not None else None, _shape(shape)
    v = triot_view(data, ctypes.cast(bs, _i64p), ctypes.cast(st, _i64p) if st else _i64p(),
                   ctypes.cast(sh, _i64p))
    return v, (bs, st, sh)


def triot_embed_view(dst: triot_view, src: triot_view, d: int, dtype: int, flags: int,
                     stream: int) -> int:
    return _lib.triot_embed_view(ctypes.byref(dst), ctypes.byref(src), d, dtype, flags, stream)


def triot_apply_binary_view(c: triot_view, a: triot_view, b: triot_view, iter_shape, d: int,
                            dtype: int, op: int, stream: int) -> int:
    return _lib.triot_apply_binary_view(ctypes.byref(c), ctypes.byref(a), ctypes.byref(b),
                                        _shape(iter_shape), d, dtype, op, stream)


def triot_expected_value_offset(out: int, p: int, shape, offset, d: int, dtype: int,
                                with_mass: int, workspace: int, workspace_bytes: int,
                                stream: int) -> int:
    return _lib.triot_expected_value_offset(out, p, _shape(shape),
                                            _shape(offset) if offset is not None else None, d,
                                            dtype, with_mass, workspace, workspace_bytes, stream)


def triot_sum_rows(out: int, rows: int, nrows: int, ncols: int, stream: int) -> int:
    return _lib.triot_sum_rows(out, rows, nrows, ncols, stream)


def triot_expected_value_host(out: int, p: int, shape, offset, d: int, dtype: int,
                              with_mass: int, staging: int, staging_bytes: int,
                              stream: int) -> int:
    return _lib.triot_expected_value_host(out, p, _shape(shape),
                                          _shape(offset) if offset is not None else None, d,
                                          dtype, with_mass, staging, staging_bytes, stream)


def triot_expected_value_view(out: int, p: triot_view, d: int, dtype: int, with_mass: int,
                              workspace: int, workspace_bytes: int, stream: int) -> int:
    return _lib.triot_expected_value_view(out, ctypes.byref(p), d, dtype, with_mass, workspace,
                                          workspace_bytes, stream)


def triot_inner_product_workspace_size() -> int:
    out = ctypes.c_size_t(0)
    check(_lib.triot_inner_product_workspace_size(ctypes.byref(out)))
    return int(out.value)


def triot_inner_product(out: int, a: int, a_shape, b: int, b_shape, iter_shape, d: int,
                        dtype: int, workspace: int, workspace_bytes: int, stream: int) -> int:
    return _lib.triot_inner_product(out, a, _shape(a_shape), b, _shape(b_shape),
                                    _shape(iter_shape), d, dtype, workspace, workspace_bytes,
                                    stream)


def triot_fused_update(x: int, x_shape, y: int, y_shape, z: int, z_shape, d: int, dtype: int,
                       stream: int) -> int:
    return _lib.triot_fused_update(x, _shape(x_shape), y, _shape(y_shape), z, _shape(z_shape), d,
                                   dtype, stream)


def triot_naive_convolve(result: int, lhs: int, lhs_shape, rhs: int, rhs_shape, d: int,
                         dtype: int, stream: int) -> int:
    return _lib.triot_naive_convolve(result, lhs, _shape(lhs_shape), rhs, _shape(rhs_shape), d,
                                     dtype, stream)


def triot_embed_host(dst: int, dst_shape, src: int, src_shape, d: int, dtype: int, flags: int,
                     staging: int, staging_bytes: int, stream: int) -> int:
    return _lib.triot_embed_host(dst, _shape(dst_shape), src, _shape(src_shape), d, dtype, flags,
                                 staging, staging_bytes, stream)


def triot_apply_binary_host(c: int, a: int, a_shape, b: int, b_shape, iter_shape, d: int,
                            dtype: int, op: int, staging: int, staging_bytes: int,
                            stream: int) -> int:
    return _lib.triot_apply_binary_host(c, a, _shape(a_shape), b, _shape(b_shape),
                                        _shape(iter_shape), d, dtype, op, staging,
                                        staging_bytes, stream)


def triot_set_launch_policy(mode: int, blocks_per_sm: int = 0) -> None:
    """Tuning hook (thread-local): -1 = automatic, 0 = chunk per warp, 1 = grid stride,
    2 / 3 = EV bulk-copy pipeline, 4 = chunk per warp with a split EV reduction."""
    check(_lib.triot_set_launch_policy(mode, blocks_per_sm))


def triot_plan_describe(op: int, shapes, iter_shape, d: int, dtype: int, flags: int = 0,
                        ptr_mod32=(0, 0, 0), mode: int = 0, warps: int = 1) -> dict:
    arrs = [_shape(s) if s is not None else None for s in shapes] + [None] * (3 - len(shapes))
    ptrs = (_i64p * 3)(*[ctypes.cast(a, _i64p) if a is not None else _i64p() for a in arrs])
    mods = (ctypes.c_uint * 3)(*ptr_mod32)
    buf = ctypes.create_string_buffer(1 << 16)
    check(_lib.triot_plan_describe(op, ptrs, _shape(iter_shape), d, dtype, flags, mods, mode,
                                   warps, buf, len(buf)))
    return json.loads(buf.value.decode())


def triot_fastdiv_magic(divisor: int) -> tuple[int, int]:
    m, s = ctypes.c_uint32(0), ctypes.c_uint32(0)
    check(_lib.triot_fastdiv_magic(divisor, ctypes.byref(m), ctypes.byref(s)))
    return int(m.value), int(s.value)

