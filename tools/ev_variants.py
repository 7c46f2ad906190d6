"""Time LDG expected-value kernel variants on C3 (diagnostic; run under ncu for cold durations).

    ncu -k regex:ev_kernel --cache-control all --clock-control none \
        --metrics gpu__time_duration.sum,launch__registers_per_thread --csv \
        --log-file gpurun_out/ev_variants.csv python tools/ev_variants.py
Prints the launch order (variant, blocks per SM) on stdout."""
import ctypes
import os
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))
import ev_probe  # noqa: E402
from triot_inputs import make_inputs  # noqa: E402

VARIANTS = {0: "K2 minB4", 1: "K4 minB4", 2: "K4 minB3", 3: "K3 minB4", 4: "K8 minB2", 5: "K4 minB2",
            6: "K2 minB5", 7: "K1 minB5", 8: "K2 minB6", 9: "K1 minB6", 10: "K1 minB8"}
# --occ: each instance at the blocks per SM its register cap allows (one wave)
OCC = {0: (4,), 6: (5,), 7: (5,), 8: (6,), 9: (6,), 10: (8,)}


def main():
    L = ev_probe.build()
    L.probe_ev_variant_c3.restype = ctypes.c_int
    L.probe_ev_variant_c3.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int, ctypes.c_int,
                                                              ctypes.c_void_p]
    dev = torch.device("cuda:0")
    p = torch.from_numpy(make_inputs("C3")["p"]).to(dev)
    ref = None
    means = torch.zeros(6, dtype=torch.float64, device=dev)
    ws = torch.zeros(1 << 20, dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    occ = "--occ" in sys.argv
    for v in (OCC if occ else VARIANTS):
        for bpsm in (OCC[v] if occ else (2, 3, 4, 6)):
            for _ in range(5 if occ else 3):
                g = L.probe_ev_variant_c3(p.data_ptr(), means.data_ptr(), ws.data_ptr(), v, bpsm, s)
                assert g > 0, g
            torch.cuda.synchronize()
            m = means.cpu().numpy()
            ref = m if ref is None else ref   # every variant sums in the same per-lane order
            print(VARIANTS[v], bpsm, g, "maxdiff_vs_first", float(abs(m - ref).max()), flush=True)


if __name__ == "__main__":
    main()
