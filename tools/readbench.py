"""Single-launch read of the C3 size (134 MB) in several decompositions (diagnostic, not product).

Run under ncu for cold-cache per-launch durations:
    ncu --cache-control all --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum \
        --csv --log-file gpurun_out/readbench.csv python tools/readbench.py
Each configuration launches once after one warm-up launch; the launch order is printed to stdout.
"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import membench  # noqa: E402


def main():
    L = membench.build()
    L.mb_read_os.restype = ctypes.c_int
    L.mb_read_os.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                             ctypes.c_void_p, ctypes.c_void_p]
    dev = torch.device("cuda:0")
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    nbytes = 16 ** 6 * 8
    src = torch.ones(nbytes // 4, dtype=torch.float32, device=dev)
    part = torch.zeros(1 << 22, dtype=torch.int32, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    cfgs = []
    for th in (256, 512):
        for u in (1, 2, 4, 8, 16):
            cfgs.append((f"read_os th={th} U={u}",
                         lambda th=th, u=u: L.mb_read_os(src.data_ptr(), nbytes, th, u, part.data_ptr(), s)))
    for bpsm in (4, 8, 16, 32, 64):
        for u in (2, 4):
            cfgs.append((f"read_k bpsm={bpsm} U={u}",
                         lambda bpsm=bpsm, u=u: L.mb_read(src.data_ptr(), nbytes, sms * bpsm, 256, u,
                                                          part.data_ptr(), s)))
    for name, fn in cfgs:
        fn()
        fn()
        torch.cuda.synchronize()
        print(name, flush=True)


if __name__ == "__main__":
    main()
