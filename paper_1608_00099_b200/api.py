"""Tensor-level wrappers: shapes from tensor.shape, pointers from data_ptr(), the stream from
torch.cuda.current_stream().  Marshalling only -- the computation is the C-ABI call."""
from __future__ import annotations

import threading

from . import _lib

OPS = {"add": _lib.TRIOT_ADD, "sub": _lib.TRIOT_SUB, "mul": _lib.TRIOT_MUL,
       "div": _lib.TRIOT_DIV}

_ws_lock = threading.Lock()
_ws_cache: dict = {}


_T = None          # torch, imported on first use (the package imports without it)
_DT = {}           # torch dtype -> triot dtype code
_RAW_STREAM = None  # torch._C._cuda_getCurrentRawStream
_GET_DEV = None     # torch._C._cuda_getDevice


def _torch():
    global _T, _RAW_STREAM, _GET_DEV
    if _T is None:
        import torch
        _DT[torch.float32] = _lib.TRIOT_F32
        _DT[torch.float64] = _lib.TRIOT_F64
        _RAW_STREAM = getattr(torch._C, "_cuda_getCurrentRawStream", None)
        _GET_DEV = getattr(torch._C, "_cuda_getDevice", None)
        _T = torch
    return _T


def _dtype_code(t) -> int:
    _torch()
    code = _DT.get(t.dtype)
    if code is None:
        raise TypeError(f"triot supports float32 and float64 tensors, got {t.dtype}")
    return code


def _check_tensor(name: str, t, device=None):
    if not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor (there is no CPU path)")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous (dense row-major)")
    if device is not None and t.device != device:
        raise ValueError(f"{name} is on {t.device}, expected {device}")


class _NoSwitch:
    __slots__ = ()

    def __enter__(self):
        return None

    def __exit__(self, *a):
        return False


_NO_SWITCH = _NoSwitch()


def _device(device):
    """Make `device` current for the C call (the library sizes grids from cudaGetDevice() and
    launches on the tensor's stream): a no-op when it already is, which is the common case."""
    torch = _torch()
    idx = device.index
    if idx is None or idx == (_GET_DEV() if _GET_DEV else torch.cuda.current_device()):
        return _NO_SWITCH
    return torch.cuda.device(idx)


def _stream(device) -> int:
    torch = _torch()
    if _RAW_STREAM is not None:   # the same handle as current_stream().cuda_stream, ~1 us cheaper
        idx = device.index if device.index is not None else torch.cuda.current_device()
        return _RAW_STREAM(idx)
    return torch.cuda.current_stream(device).cuda_stream


def _fast_pair(x, y):
    """The common case of the two-operand entry points in one pass: both contiguous CUDA tensors
    of one dtype, dimension and device.  Returns (device index, dtype code, stream) or None (the
    caller then runs the full checks, which raise the precise error)."""
    _torch()
    if not (x.is_cuda and y.is_cuda and x.is_contiguous() and y.is_contiguous()):
        return None
    idx = x.get_device()            # an int: cheaper than comparing torch.device objects
    dt = x.dtype
    code = _DT.get(dt)
    if code is None or y.dtype != dt or y.get_device() != idx or y.dim() != x.dim():
        return None
    if _RAW_STREAM is None or _GET_DEV is None or idx != _GET_DEV():
        return None
    return idx, code, _RAW_STREAM(idx)


class View:
    """A window of a dense CUDA tensor: view[t] = base[start + t].  Ops on a View
    behave as on a materialised copy of the window, without copying."""

    def __init__(self, base, start=None, shape=None):
        _check_tensor("view base", base)
        d = base.dim()
        self.base = base
        self.start = tuple(int(x) for x in (start if start is not None else (0,) * d))
        self.shape = tuple(int(x) for x in (shape if shape is not None else
                                            tuple(b - s for b, s in zip(base.shape, self.start))))
        if len(self.start) != d or len(self.shape) != d:
            raise ValueError("start and shape must have the base's dimension")

    def dim(self):
        return self.base.dim()

    def _c(self):
        return _lib.make_view(self.base.data_ptr(), tuple(self.base.shape), self.start,
                              self.shape)


def embed_view(dst: "View", src: "View", region_only: bool = False):
    """triot_embed_view: dst's window receives src's window, zero-padded."""
    if dst.base.dtype != src.base.dtype or dst.dim() != src.dim():
        raise ValueError("dst and src must have the same dtype and dimension")
    if src.base.device != dst.base.device:
        raise ValueError("dst and src must be on one device")
    (dv, keep1), (sv, keep2) = dst._c(), src._c()
    flags = _lib.TRIOT_EMBED_REGION_ONLY if region_only else _lib.TRIOT_EMBED_FULL
    with _device(dst.base.device):
        _lib.check(_lib.triot_embed_view(dv, sv, dst.dim(), _dtype_code(dst.base), flags,
                                         _stream(dst.base.device)))
    return dst


def apply_binary_view(a: "View", b: "View", out: "View", op: str = "mul", iter_shape=None):
    """triot_apply_binary_view: out_view[t] = a_view[t] OP b_view[t] over iter_shape."""
    for v in (a, b, out):
        if v.base.dtype != a.base.dtype or v.dim() != a.dim():
            raise ValueError("views must share dtype and dimension")
        if v.base.device != a.base.device:
            raise ValueError("views must be on one device")
    (cv, k1), (av, k2), (bv, k3) = out._c(), a._c(), b._c()
    with _device(a.base.device):
        _lib.check(_lib.triot_apply_binary_view(cv, av, bv, iter_shape, a.dim(),
                                                _dtype_code(a.base), OPS[op],
                                                _stream(a.base.device)))
    return out


def expected_value_view(p: "View", out=None, with_mass: bool = False):
    """triot_expected_value_view: means[k] = sum_t t_k * p_view[t] over the window (t relative
    to its start); (d+1,) with the window's mass last when with_mass."""
    torch = _torch()
    code = _dtype_code(p.base)
    d = p.dim()
    n = d + (1 if with_mass else 0)
    if out is None:
        out = torch.empty(n, dtype=torch.float64, device=p.base.device)
    _check_tensor("out", out, p.base.device)
    if out.dtype != torch.float64 or out.numel() < n:
        raise ValueError(f"out must be a float64 tensor of >= {n} elements")
    ws = workspace(tuple(p.shape), code, p.base.device)
    pv, keep = p._c()
    with _device(p.base.device):
        _lib.check(_lib.triot_expected_value_view(out.data_ptr(), pv, d, code, 1 if with_mass else 0,
                                                  ws.data_ptr(), ws.numel(),
                                                  _stream(p.base.device)))
    return out


def embed(dst, src, region_only: bool = False):
    """dst[t] = src[t] where t < src.shape, +0.0 elsewhere (or only the overlap if
    region_only).  In place on dst; returns dst."""
    fast = _fast_pair(dst, src)
    if fast is not None:   # the tensors are on the current device: no guard needed
        st = _lib._lib.triot_embed(dst.data_ptr(), _lib._shape(dst.shape), src.data_ptr(),
                                   _lib._shape(src.shape), dst.dim(), fast[1],
                                   _lib.TRIOT_EMBED_REGION_ONLY if region_only else 0, fast[2])
        if st:
            _lib.check(st)
        return dst
    dev = dst.device
    _check_tensor("dst", dst)
    _check_tensor("src", src, dev)
    if src.dtype != dst.dtype or src.dim() != dst.dim():
        raise ValueError("dst and src must have the same dtype and dimension")
    flags = _lib.TRIOT_EMBED_REGION_ONLY if region_only else _lib.TRIOT_EMBED_FULL
    with _device(dev):
        st = _lib.lib().triot_embed(dst.data_ptr(), _lib._shape(dst.shape), src.data_ptr(),
                                    _lib._shape(src.shape), dst.dim(), _dtype_code(dst), flags,
                                    _stream(dev))
    if st:
        _lib.check(st)
    return dst


class Prepared:
    """A call with its arguments marshalled once (P:266 calls the dispatch "already a prerequisite
    cost"; for a 75 KB op the Python-side marshalling is most of the time per call).  Calling the
    object re-issues the same C-ABI call -- same tensors, same shapes -- on the device's current
    stream; the tensors are kept alive by it.  Marshalling only, as the plain wrappers."""
    __slots__ = ("_fn", "_args", "_idx", "_keep", "result")

    def __init__(self, fn, args, idx, keep, result):
        self._fn, self._args, self._idx, self._keep, self.result = fn, args, idx, keep, result

    def __call__(self):
        if _GET_DEV is not None and _RAW_STREAM is not None and _GET_DEV() == self._idx:
            st = self._fn(*self._args, _RAW_STREAM(self._idx))
        else:
            with _device(self.result.device):
                st = self._fn(*self._args, _stream(self.result.device))
        if st:
            _lib.check(st)
        return self.result


def prepare_embed(dst, src, region_only: bool = False) -> Prepared:
    """embed(dst, src, region_only) as a re-issuable call: checks and argument marshalling
    happen here, once; each call of the result is one triot_embed."""
    _torch()
    _check_tensor("dst", dst)
    _check_tensor("src", src, dst.device)
    if src.dtype != dst.dtype or src.dim() != dst.dim():
        raise ValueError("dst and src must have the same dtype and dimension")
    import ctypes
    flags = _lib.TRIOT_EMBED_REGION_ONLY if region_only else _lib.TRIOT_EMBED_FULL
    args = (ctypes.c_void_p(dst.data_ptr()), _lib._shape(tuple(dst.shape)),
            ctypes.c_void_p(src.data_ptr()), _lib._shape(tuple(src.shape)), dst.dim(),
            _dtype_code(dst), flags)
    return Prepared(_lib.lib().triot_embed, args, dst.get_device(), (dst, src), dst)


def prepare_apply_binary(a, b, op: str = "mul", out=None, iter_shape=None) -> Prepared:
    """apply_binary(a, b, op, out, iter_shape) as a re-issuable call (see prepare_embed)."""
    torch = _torch()
    _check_tensor("a", a)
    _check_tensor("b", b, a.device)
    if a.dtype != b.dtype or a.dim() != b.dim():
        raise ValueError("a and b must have the same dtype and dimension")
    if iter_shape is None:
        iter_shape = tuple(min(x, y) for x, y in zip(a.shape, b.shape))
    iter_shape = tuple(int(x) for x in iter_shape)
    if out is None:
        out = torch.empty(iter_shape, dtype=a.dtype, device=a.device)
    _check_tensor("out", out, a.device)
    if out.dtype != a.dtype or out.dim() != a.dim():
        raise ValueError("out must have the operands' dtype and dimension")
    import ctypes
    args = (ctypes.c_void_p(out.data_ptr()), _lib._shape(tuple(out.shape)),
            ctypes.c_void_p(a.data_ptr()), _lib._shape(tuple(a.shape)),
            ctypes.c_void_p(b.data_ptr()), _lib._shape(tuple(b.shape)), _lib._shape(iter_shape),
            a.dim(), _dtype_code(a), OPS[op])
    return Prepared(_lib.lib().triot_apply_binary, args, a.get_device(), (a, b, out), out)


def apply_binary(a, b, op: str = "mul", out=None, iter_shape=None):
    """out[t] = a[t] OP b[t] for t in iter_shape (default: element-wise min of the shapes).
    `out` defaults to a new tensor dense in iter_shape."""
    torch = _torch()
    fast = _fast_pair(a, b)
    if fast is not None and out is not None and iter_shape is None and out.is_cuda and \
            out.is_contiguous() and out.dtype == a.dtype and out.get_device() == fast[0]:
        st = _lib._lib.triot_apply_binary(out.data_ptr(), _lib._shape(out.shape), a.data_ptr(),
                                          _lib._shape(a.shape), b.data_ptr(),
                                          _lib._shape(b.shape), None, a.dim(), fast[1],
                                          OPS[op], fast[2])
        if st:
            _lib.check(st)
        return out
    _check_tensor("a", a)
    _check_tensor("b", b, a.device)
    if a.dtype != b.dtype or a.dim() != b.dim():
        raise ValueError("a and b must have the same dtype and dimension")
    if iter_shape is None:
        iter_shape = tuple(min(x, y) for x, y in zip(a.shape, b.shape))
    iter_shape = tuple(int(x) for x in iter_shape)
    if out is None:
        out = torch.empty(iter_shape, dtype=a.dtype, device=a.device)
    _check_tensor("out", out, a.device)
    if out.dtype != a.dtype:
        raise ValueError("out must have the dtype of a and b")
    with _device(a.device):
        _lib.check(_lib.triot_apply_binary(out.data_ptr(), tuple(out.shape), a.data_ptr(),
                                           tuple(a.shape), b.data_ptr(), tuple(b.shape), iter_shape,
                                           a.dim(), _dtype_code(a), OPS[op], _stream(a.device)))
    return out


def workspace(p_shape, dtype_code: int, device):
    """The cached, once-zeroed expected-value workspace for (device, current stream)."""
    torch = _torch()
    need = _lib.triot_expected_value_workspace_size(tuple(p_shape), len(p_shape), dtype_code)
    key = (device, _stream(device))
    with _ws_lock:
        ws = _ws_cache.get(key)
        if ws is None or ws.numel() < need:
            ws = torch.zeros(need, dtype=torch.uint8, device=device)
            _ws_cache[key] = ws
    return ws


def expected_value(p, out=None, with_mass: bool = False, offset=None):
    """means[k] = sum_t t_k * p[t] (fp64), k = 0..d-1.  Returns a (d,) float64 CUDA tensor, or
    (d+1,) with out[d] = sum_t p[t] when with_mass (triot_expected_value_mass).  offset: p is
    the block of a larger PMF whose element t sits at offset + t; the weights are then the
    global coordinates (triot_expected_value_offset, P:607 slabs)."""
    torch = _torch()
    _check_tensor("p", p)
    code = _dtype_code(p)
    d = p.dim()
    n = d + (1 if with_mass else 0)
    if out is None:
        out = torch.empty(n, dtype=torch.float64, device=p.device)
    _check_tensor("out", out, p.device)
    if out.dtype != torch.float64 or out.numel() < n:
        raise ValueError(f"out must be a float64 tensor of >= {n} elements")
    ws = workspace(tuple(p.shape), code, p.device)
    with _device(p.device):
        if offset is not None:
            off = tuple(int(x) for x in offset)
            if len(off) != d:
                raise ValueError(f"offset must have {d} entries")
            _lib.check(_lib.triot_expected_value_offset(
                out.data_ptr(), p.data_ptr(), tuple(p.shape), off, d, code,
                1 if with_mass else 0, ws.data_ptr(), ws.numel(), _stream(p.device)))
        else:
            fn = _lib.triot_expected_value_mass if with_mass else _lib.triot_expected_value
            _lib.check(fn(out.data_ptr(), p.data_ptr(), tuple(p.shape), d, code, ws.data_ptr(),
                          ws.numel(), _stream(p.device)))
    return out


def sum_rows(rows, out=None):
    """out[j] = sum_r rows[r, j], rows added in order (triot_sum_rows): the deterministic
    amalgamation of per-slab / per-rank results.  rows: a 2-D float64 CUDA tensor."""
    torch = _torch()
    _check_tensor("rows", rows)
    if rows.dtype != torch.float64 or rows.dim() != 2:
        raise ValueError("rows must be a 2-D float64 tensor")
    nr, nc = int(rows.shape[0]), int(rows.shape[1])
    if out is None:
        out = torch.empty(nc, dtype=torch.float64, device=rows.device)
    _check_tensor("out", out, rows.device)
    with _device(rows.device):
        _lib.check(_lib.triot_sum_rows(out.data_ptr(), rows.data_ptr(), nr, nc,
                                       _stream(rows.device)))
    return out


def expected_value_host(p, staging=None, out=None, with_mass: bool = False, offset=None,
                        device=None):
    """triot_expected_value_host: the expected value of a (pinned) host tensor p, streamed in
    chunks through the device `staging` buffer (a uint8 CUDA tensor, 256-byte aligned); returns
    a host float64 tensor (pinned when allocated here), valid once the current stream has
    completed.  offset: p is the block at that tuple of a larger PMF (global weights)."""
    torch = _torch()
    if p.is_cuda or not p.is_contiguous():
        raise ValueError("p must be a contiguous host tensor")
    code = _dtype_code(p)
    d = p.dim()
    n = d + (1 if with_mass else 0)
    if out is None:
        out = torch.empty(n, dtype=torch.float64, pin_memory=True)
    if staging is None:
        dev = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        staging = globals()["staging"](dev)
    dev = staging.device
    with _device(dev):
        off = tuple(int(x) for x in offset) if offset is not None else None
        _lib.check(_lib.triot_expected_value_host(out.data_ptr(), p.data_ptr(), tuple(p.shape),
                                                  off, d, code, 1 if with_mass else 0,
                                                  staging.data_ptr(), staging.numel(),
                                                  _stream(dev)))
    return out


def inner_product(a, b, iter_shape=None, out=None):
    """Benchmark 2 / Alg 8 dot_product: sum_t a[t] * b[t] over iter_shape (default: the shared
    tuples).  Returns a (1,) float64 CUDA tensor."""
    torch = _torch()
    _check_tensor("a", a)
    _check_tensor("b", b, a.device)
    if a.dtype != b.dtype or a.dim() != b.dim():
        raise ValueError("a and b must have the same dtype and dimension")
    if out is None:
        out = torch.empty(1, dtype=torch.float64, device=a.device)
    need = _lib.triot_inner_product_workspace_size()
    key = ("dot", a.device, _stream(a.device))
    with _ws_lock:
        ws = _ws_cache.get(key)
        if ws is None or ws.numel() < need:
            ws = torch.zeros(need, dtype=torch.uint8, device=a.device)
            _ws_cache[key] = ws
    with _device(a.device):
        _lib.check(_lib.triot_inner_product(out.data_ptr(), a.data_ptr(), tuple(a.shape),
                                            b.data_ptr(), tuple(b.shape), iter_shape, a.dim(),
                                            _dtype_code(a), ws.data_ptr(), ws.numel(),
                                            _stream(a.device)))
    return out


def fused_update(x, y, z):
    """Benchmark 3: x[t] = x[t] + y[t]*x[t] - z[t] over x's shape, in place; returns x."""
    _check_tensor("x", x)
    _check_tensor("y", y, x.device)
    _check_tensor("z", z, x.device)
    if not (x.dtype == y.dtype == z.dtype) or not (x.dim() == y.dim() == z.dim()):
        raise ValueError("x, y, z must share dtype and dimension")
    with _device(x.device):
        _lib.check(_lib.triot_fused_update(x.data_ptr(), tuple(x.shape), y.data_ptr(), tuple(y.shape),
                                           z.data_ptr(), tuple(z.shape), x.dim(), _dtype_code(x),
                                           _stream(x.device)))
    return x


def naive_convolve(lhs, rhs, out=None):
    """Alg 15 (Benchmark 4): result[t_l + t_r] += lhs[t_l] * rhs[t_r], shape lhs + rhs - 1."""
    torch = _torch()
    _check_tensor("lhs", lhs)
    _check_tensor("rhs", rhs, lhs.device)
    if lhs.dtype != rhs.dtype or lhs.dim() != rhs.dim():
        raise ValueError("lhs and rhs must have the same dtype and dimension")
    shape = tuple(a + b - 1 for a, b in zip(lhs.shape, rhs.shape))
    if out is None:
        out = torch.empty(shape, dtype=lhs.dtype, device=lhs.device)
    _check_tensor("out", out, lhs.device)
    if tuple(out.shape) != shape or out.dtype != lhs.dtype:
        raise ValueError(f"out must be {lhs.dtype} of shape {shape}")
    with _device(lhs.device):
        _lib.check(_lib.triot_naive_convolve(out.data_ptr(), lhs.data_ptr(), tuple(lhs.shape),
                                             rhs.data_ptr(), tuple(rhs.shape), lhs.dim(),
                                             _dtype_code(lhs), _stream(lhs.device)))
    return out


# ---- host buffers: chunked streaming through a device staging buffer ----------------

STAGING_BYTES = 256 << 20


def staging(device, nbytes: int | None = None):
    """The cached device staging buffer for (device, current stream)."""
    torch = _torch()
    nbytes = STAGING_BYTES if nbytes is None else nbytes
    key = ("staging", device, _stream(device))
    with _ws_lock:
        buf = _ws_cache.get(key)
        if buf is None or buf.numel() != nbytes:
            buf = torch.empty(nbytes, dtype=torch.uint8, device=device)
            _ws_cache[key] = buf
    return buf


def _check_host(name, t):
    if t.is_cuda or not t.is_contiguous():
        raise TypeError(f"{name} must be a contiguous host (CPU) tensor; pin it for overlap")


def embed_host(dst, src, device=None):
    """embed on HOST tensors (pinned for full overlap): slabs of dst's axis 0 are streamed
    through device staging memory (H2D / kernel / D2H overlapped).  Asynchronous: synchronize
    the current stream before reading dst."""
    torch = _torch()
    _check_host("dst", dst)
    _check_host("src", src)
    if src.dtype != dst.dtype or src.dim() != dst.dim():
        raise ValueError("dst and src must have the same dtype and dimension")
    device = torch.device(device) if device is not None else torch.device(
        "cuda", torch.cuda.current_device())
    buf = staging(device)
    with torch.cuda.device(device):
        _lib.check(_lib.triot_embed_host(dst.data_ptr(), tuple(dst.shape), src.data_ptr(),
                                         tuple(src.shape), dst.dim(), _dtype_code(dst),
                                         _lib.TRIOT_EMBED_FULL, buf.data_ptr(), buf.numel(),
                                         _stream(device)))
    return dst


def apply_binary_host(a, b, op: str = "mul", out=None, iter_shape=None, device=None):
    """apply_binary on HOST tensors; out (host, dense in iter_shape) is created pinned if None."""
    torch = _torch()
    _check_host("a", a)
    _check_host("b", b)
    if iter_shape is None:
        iter_shape = tuple(min(x, y) for x, y in zip(a.shape, b.shape))
    iter_shape = tuple(int(x) for x in iter_shape)
    if out is None:
        out = torch.empty(iter_shape, dtype=a.dtype).pin_memory()
    _check_host("out", out)
    device = torch.device(device) if device is not None else torch.device(
        "cuda", torch.cuda.current_device())
    buf = staging(device)
    with torch.cuda.device(device):
        _lib.check(_lib.triot_apply_binary_host(out.data_ptr(), a.data_ptr(), tuple(a.shape),
                                                b.data_ptr(), tuple(b.shape), iter_shape,
                                                a.dim(), _dtype_code(a), OPS[op], buf.data_ptr(),
                                                buf.numel(), _stream(device)))
    return out
