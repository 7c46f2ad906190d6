"""C3 expected value: the dedicated-reducer-block reduction vs the ticket tail (diagnostic).
Probe entry probe_ev_rb_c3: `git apply tools/dbg/ev_r02_reducer_block.patch` first (measured, not kept:
profiles/r02_ev11_reducer_block*).

    python tools/ev_rb.py                 # events: single (L2 flushed) + 20 back to back in a graph
    ncu --cache-control all --clock-control none --metrics gpu__time_duration.sum --csv \
        --log-file gpurun_out/ev_rb.csv python tools/ev_rb.py --ncu
Prints one JSON line per configuration (launch order = line order under --ncu)."""
import ctypes
import json
import os
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))
import ev_probe  # noqa: E402
import membench  # noqa: E402
from triot_inputs import make_inputs  # noqa: E402

VARIANTS = {0: "K2 ticket", 1: "K2 reducer block"}


def main():
    ncu = "--ncu" in sys.argv
    L = ev_probe.build()
    L.probe_ev_rb_c3.restype = ctypes.c_int
    L.probe_ev_rb_c3.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int, ctypes.c_int,
                                                            ctypes.c_void_p]
    M = membench.build()
    dev = torch.device("cuda:0")
    import paper_1608_00099_b200 as T
    p = torch.from_numpy(make_inputs("C3")["p"]).to(dev)
    ref = T.expected_value(p).cpu()
    means = torch.zeros(6, dtype=torch.float64, device=dev)
    ws = torch.zeros(1 << 20, dtype=torch.uint8, device=dev)
    part = torch.zeros(1 << 22, dtype=torch.int32, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    clean = torch.ones(256 << 20, dtype=torch.int32, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    nbytes = p.numel() * 8

    def timed(fn):
        if ncu:
            fn(); fn()
            torch.cuda.synchronize()
            return {}
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        single = []
        for _ in range(30):
            flush.fill_(1)
            clean.sum()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); fn(); b.record()
            torch.cuda.synchronize()
            single.append(a.elapsed_time(b) * 1000)
        single.sort()
        g = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            fn()
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=st):
                for _ in range(20):
                    fn()
        g.replay(); torch.cuda.synchronize()
        b2b = []
        for _ in range(10):
            flush.fill_(1)
            clean.sum()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); g.replay(); b.record()
            torch.cuda.synchronize()
            b2b.append(a.elapsed_time(b) * 1000 / 20)
        b2b.sort()
        return {"single_us": round(single[len(single) // 2], 2),
                "single_min_us": round(single[0], 2), "b2b_us": round(b2b[len(b2b) // 2], 2)}

    for bpsm in (8, 16):
        r = timed(lambda bpsm=bpsm: M.mb_read(p.data_ptr(), nbytes, sms * bpsm, 256, 4,
                                              part.data_ptr(), torch.cuda.current_stream().cuda_stream))
        print(json.dumps({"kind": "read134MB", "bpsm": bpsm, **r}), flush=True)
    r = timed(lambda: T.expected_value(p, out=means))
    print(json.dumps({"kind": "library", **r}), flush=True)
    for v in VARIANTS:
        for bpsm in (4, 8, 16):
            grid = [0]

            def fn(v=v, bpsm=bpsm):
                grid[0] = L.probe_ev_rb_c3(p.data_ptr(), means.data_ptr(), ws.data_ptr(), v, bpsm,
                                              torch.cuda.current_stream().cuda_stream)
                assert grid[0] > 0, grid[0]
            fn(); torch.cuda.synchronize()
            m1 = means.cpu()
            fn(); torch.cuda.synchronize()
            m2 = means.cpu()
            det = bool(torch.equal(m1, m2))
            rel = float(((m1 - ref).abs() / ref.abs()).max())
            r = timed(fn)
            print(json.dumps({"kind": "exact", "variant": VARIANTS[v], "bpsm": bpsm, "grid": grid[0],
                              "det": det, "rel_vs_lib": rel, **r}), flush=True)


if __name__ == "__main__":
    main()
