"""PCIe copy ceilings for the e2e leg (diagnostic): pinned H2D, D2H, and both at once.

    python tools/pcie_probe.py > gpurun_out/pcie.jsonl
"""
import json

import torch


def main():
    dev = torch.device("cuda:0")
    n = 1 << 30
    h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
    d_a = torch.empty(n, dtype=torch.uint8, device=dev)
    d_b = torch.empty(n, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream()
        a.record(cur)
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        fn()
        cur.wait_stream(s1)
        cur.wait_stream(s2)
        b.record(cur)
        torch.cuda.synchronize()
        return a.elapsed_time(b) * 1e-3

    def h2d():
        with torch.cuda.stream(s1):
            d_a.copy_(h_in, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            h_out.copy_(d_b, non_blocking=True)

    def both():
        h2d()
        d2h()

    for name, fn, moved in (("h2d", h2d, n), ("d2h", d2h, n), ("both", both, 2 * n)):
        t = timed(fn)
        print(json.dumps({"copy": name, "GB": moved / 1e9, "s": round(t, 5),
                          "GBps": round(moved / t / 1e9, 2)}), flush=True)


if __name__ == "__main__":
    main()
