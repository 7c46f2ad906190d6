"""Host cost per call of the C1 embed through each layer (diagnostic): the Python wrapper, the
raw ctypes call with prebuilt arguments, and a one-element torch fill, wall clock over many
back-to-back calls (the GPU keeps up: ~1.6 us per op)."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1608_00099_b200 as T  # noqa: E402
from paper_1608_00099_b200 import _lib  # noqa: E402


def per_call(fn, n=20000):
    for _ in range(200):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / n * 1e6


def main():
    dev = torch.device("cuda:0")
    src = torch.rand((4, 9, 7, 5), dtype=torch.float64, device=dev)
    dst = torch.empty((8, 16, 8, 8), dtype=torch.float64, device=dev)
    z = torch.empty(1, dtype=torch.float64, device=dev)
    raw = _lib.lib().triot_embed
    ds, ss = _lib._shape(dst.shape), _lib._shape(src.shape)
    dp, sp = dst.data_ptr(), src.data_ptr()
    stream = torch.cuda.current_stream().cuda_stream
    res = {
        "api_embed": per_call(lambda: T.embed(dst, src)),
        "raw_ctypes_embed": per_call(lambda: raw(dp, ds, sp, ss, 4, 1, 0, stream)),
        "torch_fill_1elem": per_call(lambda: z.fill_(0.0)),
        "python_noop_lambda": per_call(lambda: None),
    }
    print(json.dumps({k: round(v, 3) for k, v in res.items()}))


if __name__ == "__main__":
    main()
