"""Sweep the work-decomposition policy per BASELINE config (tuning tool, B200).

    python tools/tune.py [--only C2,C5] > gpurun_out/tune.jsonl

For each op: mode 0 (chunk per warp) / 1 (grid stride) x blocks per SM, timed as one launch
after an L2 scrub and as the mean of 20 back-to-back launches (CUDA events).  The winners are
baked into capi.cu's auto_policy(); DESIGN.md §Decomposition records the table.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1608_00099_b200 as T  # noqa: E402
from bench import algorithmic_bytes  # noqa: E402
from triot_inputs import make_inputs  # noqa: E402


def op_fn(name, dev):
    inp = make_inputs(name)
    if name in ("C1", "C2", "C5"):
        src = torch.from_numpy(inp["src"]).to(dev)
        dst = torch.empty(inp["dst_shape"], dtype=src.dtype, device=dev)
        return lambda: T.embed(dst, src)
    if name == "C3":
        p = torch.from_numpy(inp["p"]).to(dev)
        out = torch.empty(p.dim(), dtype=torch.float64, device=dev)
        return lambda: T.expected_value(p, out=out)
    a = torch.from_numpy(inp["a"]).to(dev)
    b = torch.from_numpy(inp["b"]).to(dev)
    c = torch.empty(inp["iter_shape"], dtype=torch.float64, device=dev)
    return lambda: T.apply_binary(a, b, "mul", out=c)


def timeit(fn, scrub, reps=20):
    st = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    singles = []
    for _ in range(9):
        scrub()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        singles.append(a.elapsed_time(b))
    a.record(st)
    for _ in range(reps):
        fn()
    b.record(st)
    torch.cuda.synchronize()
    return sum(singles) / len(singles), a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="C1,C2,C3,C4,C5")
    ap.add_argument("--bpsm", default="0,1,2,3,4,6,8,12,16")
    ap.add_argument("--modes", default="0,1")
    ap.add_argument("--membench", action="store_true")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    scratch = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    clean = torch.ones(512 << 18, dtype=torch.int32, device=dev)

    def scrub():
        # evict everything and leave the L2 clean: write a buffer, then read another one (the
        # read forces the write-back of every dirty line before the timed launch)
        scratch.fill_(1)
        clean.sum()
    if a.membench:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import membench
        L = membench.build()
        src = torch.ones(134217728 // 4, dtype=torch.float32, device=dev)
        sink = torch.zeros(4, dtype=torch.int32, device=dev)
        s = torch.cuda.current_stream().cuda_stream
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        for bpsm in (2, 4, 8, 16):
            for u in (4, 8):
                single, b2b = timeit(lambda: L.mb_read(src.data_ptr(), 134217728, sms * bpsm, 256,
                                                       u, sink.data_ptr(), s), scrub)
                print(json.dumps({"config": "read134MB", "mode": -1, "bpsm": bpsm, "U": u,
                                  "single_us": round(single * 1000, 2),
                                  "b2b_us": round(b2b * 1000, 2),
                                  "single_gbs": round(134217728 / single / 1e6, 1),
                                  "b2b_gbs": round(134217728 / b2b / 1e6, 1)}), flush=True)
    for name in a.only.split(","):
        fn = op_fn(name, dev)
        nb = algorithmic_bytes(name)
        for mode in [int(x) for x in a.modes.split(",")]:
            for bpsm in [int(x) for x in a.bpsm.split(",")]:
                T.triot_set_launch_policy(mode, bpsm)
                single, b2b = timeit(fn, scrub)
                print(json.dumps({"config": name, "mode": mode, "bpsm": bpsm,
                                  "single_us": round(single * 1000, 2),
                                  "b2b_us": round(b2b * 1000, 2),
                                  "single_gbs": round(nb / single / 1e6, 1),
                                  "b2b_gbs": round(nb / b2b / 1e6, 1)}), flush=True)
        T.triot_set_launch_policy(-1, 0)


if __name__ == "__main__":
    main()
