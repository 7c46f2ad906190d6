"""Host-buffer (e2e) legs one at a time and together (diagnostic): where the e2e step's PCIe time
goes.  python tools/e2e_probe.py > gpurun_out/e2e_probe.jsonl"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1608_00099_b200 as T  # noqa: E402
from triot_inputs import make_inputs  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    h = {n: make_inputs(n) for n in ("C2", "C3", "C4", "C5")}
    src2 = torch.from_numpy(h["C2"]["src"]).pin_memory()
    p3 = torch.from_numpy(h["C3"]["p"]).pin_memory()
    a4 = torch.from_numpy(h["C4"]["a"]).pin_memory()
    b4 = torch.from_numpy(h["C4"]["b"]).pin_memory()
    src5 = torch.from_numpy(h["C5"]["src"]).pin_memory()
    dst2 = torch.empty(h["C2"]["dst_shape"], dtype=torch.float32).pin_memory()
    c4 = torch.empty(h["C4"]["iter_shape"], dtype=torch.float64).pin_memory()
    dst5 = torch.empty(h["C5"]["dst_shape"], dtype=torch.float32).pin_memory()
    m3 = torch.empty(6, dtype=torch.float64).pin_memory()
    main_s = torch.cuda.current_stream()
    side = [torch.cuda.Stream(dev) for _ in range(4)]
    legs = {
        "C2": lambda: T.embed_host(dst2, src2, device=dev),
        "C3": lambda: T.expected_value_host(p3, out=m3, device=dev),
        "C4": lambda: T.apply_binary_host(a4, b4, "mul", out=c4, device=dev),
        "C5": lambda: T.embed_host(dst5, src5, device=dev),
    }

    def run(names):
        for i, n in enumerate(names):
            side[i].wait_stream(main_s)
            with torch.cuda.stream(side[i]):
                legs[n]()
        for i in range(len(names)):
            main_s.wait_stream(side[i])

    def timed(names, reps=3):
        run(names)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(main_s)
        for _ in range(reps):
            run(names)
        b.record(main_s)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    slots = os.environ.get("TRIOT_HOST_SLOTS", "2")
    order = ["C5", "C2", "C4", "C3"]
    if os.environ.get("E2E_ORDER_ONLY"):
        ms = [round(timed(order, reps=4), 3) for _ in range(3)]
        print(json.dumps({"slots": slots, "legs": order, "ms": ms}), flush=True)
        return
    for names in (["C2", "C3", "C4", "C5"], order):
        print(json.dumps({"slots": slots, "staging_MB": T.api.STAGING_BYTES >> 20, "legs": names,
                          "ms": round(timed(names), 3)}), flush=True)
    for mb in (128, 512):
        T.api.STAGING_BYTES = mb << 20
        T.api._ws_cache.clear()
        print(json.dumps({"slots": slots, "staging_MB": mb, "legs": "all",
                          "ms": round(timed(["C2", "C3", "C4", "C5"]), 3)}), flush=True)


if __name__ == "__main__":
    main()
