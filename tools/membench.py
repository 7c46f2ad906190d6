"""HBM ceilings on this B200 for the traffic mixes of the TRIOT ops (diagnostic, not product).

    python tools/membench.py > gpurun_out/membench.json

Builds tools/libmembench.so (nvcc, sm_100a) on first use.  Each line: kernel, geometry, GB/s
(read+write bytes / CUDA-event time), once after an L2 scrub and as the mean of 10
back-to-back launches.
"""
import ctypes
import json
import os
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libmembench.so")


def build():
    src = os.path.join(HERE, "membench.cu")
    if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(src):
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                        "-Xcompiler", "-fPIC", "-o", SO, src], check=True)
    L = ctypes.CDLL(SO)
    for f in ("mb_write", "mb_read", "mb_mix", "mb_write_gs", "mb_mix_gs", "mb_mix_bc",
              "mb_write_os", "mb_write_occ"):
        getattr(L, f).restype = ctypes.c_int
    L.mb_write.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                           ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
    L.mb_read.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                          ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    L.mb_mix.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int,
                         ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
    L.mb_write_gs.argtypes = L.mb_write.argtypes
    L.mb_mix_gs.argtypes = L.mb_mix.argtypes
    L.mb_mix_bc.argtypes = L.mb_mix.argtypes
    L.mb_write_occ.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                               ctypes.c_int, ctypes.c_void_p]
    L.mb_write_os.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                              ctypes.c_int, ctypes.c_void_p]
    return L


def timeit(fn, scrub, reps=10):
    st = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    scrub()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    fn()
    b.record(st)
    torch.cuda.synchronize()
    single = a.elapsed_time(b)
    a.record(st)
    for _ in range(reps):
        fn()
    b.record(st)
    torch.cuda.synchronize()
    return single, a.elapsed_time(b) / reps


def main():
    L = build()
    dev = torch.device("cuda:0")
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    nbytes = 1 << 30
    src = torch.ones(nbytes // 4, dtype=torch.float32, device=dev)
    dst = torch.empty(nbytes // 4, dtype=torch.float32, device=dev)
    scratch = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    sink = torch.zeros(4, dtype=torch.int32, device=dev)
    scrub = lambda: scratch.fill_(1)
    s = torch.cuda.current_stream().cuda_stream
    out = []

    def rec(kind, geom, moved, t):
        out.append({"kind": kind, "geom": geom, "single_gbs": round(moved / t[0] / 1e6, 1),
                    "b2b_gbs": round(moved / t[1] / 1e6, 1)})
        print(json.dumps(out[-1]), flush=True)

    rec("torch.fill_", "", nbytes, timeit(lambda: dst.fill_(0.0), scrub))
    if "--occ" in sys.argv:
        for smem, nb in ((0, 8), (36 << 10, 6), (44 << 10, 5), (54 << 10, 4), (72 << 10, 3), (110 << 10, 2)):
            for bpsm in (64, 128):
                rec("write_occ", f"blocks/SM={nb} bpsm={bpsm}", nbytes,
                    timeit(lambda: L.mb_write_occ(dst.data_ptr(), nbytes, sms * bpsm, 256, smem, s), scrub))
        return
    if "--os" in sys.argv:
        for vb in (16, 32):
            for th in (128, 256, 512):
                for u in (1, 2, 4, 8):
                    rec("write_os", f"vb={vb} threads={th} U={u}", nbytes,
                        timeit(lambda: L.mb_write_os(dst.data_ptr(), nbytes, vb, th, u, s), scrub))
        for bpsm in (8, 16, 32, 64):
            rec("write", f"bpsm={bpsm} pol=1 U=4", nbytes,
                timeit(lambda: L.mb_write(dst.data_ptr(), nbytes, sms * bpsm, 256, 1, 4, s), scrub))
        rec("torch.fill_", "again", nbytes, timeit(lambda: dst.fill_(0.0), scrub))
        return
    if "--gs" in sys.argv:
        for bpsm in (2, 4, 8, 16):
            for pol in (0, 2):
                for u in (1, 4):
                    rec("write_gs", f"bpsm={bpsm} pol={pol} U={u}", nbytes,
                        timeit(lambda: L.mb_write_gs(dst.data_ptr(), nbytes, sms * bpsm, 256, pol, u, s), scrub))
        for rd in (64, 27, 1):
            for bpsm in (2, 4, 8):
                for u in (1, 2, 4):
                    moved = nbytes + nbytes * rd // 64
                    rec(f"mix_gs rd={rd}/64", f"bpsm={bpsm} U={u}", moved,
                        timeit(lambda: L.mb_mix_gs(src.data_ptr(), dst.data_ptr(), nbytes, sms * bpsm, 256, u, rd, s), scrub))
                    if u > 1:
                        rec(f"mix_bc rd={rd}/64", f"bpsm={bpsm} U={u}", moved,
                            timeit(lambda: L.mb_mix_bc(src.data_ptr(), dst.data_ptr(), nbytes, sms * bpsm, 256, u, rd, s), scrub))
        return
    rec("torch.copy_", "", 2 * nbytes, timeit(lambda: dst.copy_(src), scrub))
    for bpsm in (2, 4, 8):
        for pol in (0, 1, 2, 3):
            for u in (4, 8):
                rec("write", f"bpsm={bpsm} pol={pol} U={u}", nbytes,
                    timeit(lambda: L.mb_write(dst.data_ptr(), nbytes, sms * bpsm, 256, pol, u, s),
                           scrub))
    for bpsm in (2, 4, 8):
        for u in (2, 4, 8):
            rec("read", f"bpsm={bpsm} U={u}", nbytes,
                timeit(lambda: L.mb_read(src.data_ptr(), nbytes, sms * bpsm, 256, u,
                                         sink.data_ptr(), s), scrub))
    for rd in (64, 27, 1):
        for bpsm in (2, 4, 8):
            for u in (2, 4):
                moved = nbytes + nbytes * rd // 64
                rec(f"mix rd={rd}/64", f"bpsm={bpsm} U={u}", moved,
                    timeit(lambda: L.mb_mix(src.data_ptr(), dst.data_ptr(), nbytes, sms * bpsm,
                                            256, u, rd, s), scrub))


if __name__ == "__main__":
    main()
