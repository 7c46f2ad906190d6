"""Per-op time of launch-bound kernels in a CUDA graph (diagnostic; builds tools/liblatprobe.so).
    python tools/latency_probe.py"""
import ctypes
import json
import os
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
DEFS = os.environ.get("LATPROBE_DEFS", "").split()   # e.g. "-DTRIOT_ONESTEP=0": A/B
SO = os.path.join(HERE, "liblatprobe%s.so" % ("_" + "".join(c for c in "".join(DEFS) if c.isalnum()) if DEFS else ""))


def build():
    srcs = [os.path.join(HERE, "latency_probe.cu"),
            os.path.join(ROOT, "paper_1608_00099_b200", "csrc", "plan.cpp")]
    if not os.path.exists(SO) or any(os.path.getmtime(x) > os.path.getmtime(SO) for x in srcs):
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                        "-shared", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"), *DEFS,
                        "-o", SO, *srcs], check=True)
    L = ctypes.CDLL(SO)
    L.probe_latency.restype = ctypes.c_double
    L.probe_latency.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_int]
    return L


def main():
    L = build()
    dev = torch.device("cuda:0")
    dst = torch.empty((8, 16, 8, 8), dtype=torch.float64, device=dev)
    src = torch.rand((4, 9, 7, 5), dtype=torch.float64, device=dev)
    scratch = torch.zeros(65536, dtype=torch.float64, device=dev)
    names = ["empty+pdl", "empty plain", "1 load+1 store, pdl", "C1 embed 8 blocks pdl",
             "C1 embed 1 block pdl", "C1 embed 8 blocks no pdl", "copy 8x256x4 pdl",
             "copy 8x256x4 with 1.3 KB descriptor, pdl"]
    names = list(enumerate(names)) + [(9, "binary mul (9,16,8,8)x(8,17,8,8)->(8,16,8,8) 8 blocks pdl"), (10, "copy 64 KB, 32-B vector per thread, 8x256"),
                                      (11, "same, 16x128"), (12, "same, 32x64"), (13, "same, 64x32"),
                                      (14, "stores only, 8x256"), (15, "loads only, 8x256")]
    for v, nm in names:
        us = [L.probe_latency(v, dst.data_ptr(), src.data_ptr(), scratch.data_ptr(), 200)
              for _ in range(3)]
        print(json.dumps({"variant": nm, "us_per_op": [round(x, 3) for x in us]}), flush=True)


if __name__ == "__main__":
    main()
