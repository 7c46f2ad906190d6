"""Run each TRIOT op on its BASELINE config a few times (profiling driver for ncu).

    python tools/profile_ops.py [--only C5] [--reps 3]

Every launch is one of the library's kernels; inputs are built before the first launch.
Exits 0 only if every op ran (no parity check here -- that is tests/)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1608_00099_b200 as T  # noqa: E402
from triot_inputs import make_inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="C1,C2,C3,C4,C5")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--policy", default=None, help="mode,blocks_per_sm (triot_set_launch_policy)")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    if a.policy:
        mode, bpsm = (int(x) for x in a.policy.split(","))
        T.triot_set_launch_policy(mode, bpsm)
    for name in a.only.split(","):
        if name in ("B4", "CONVBIG"):
            import numpy as np
            rng = np.random.default_rng(17)
            sh = (256, 8) if name == "B4" else (48, 48, 8)   # CONVBIG: 135k outputs, 340M MACs
            l4 = torch.from_numpy(rng.random(sh)).to(dev)
            r4 = torch.from_numpy(rng.random(sh)).to(dev)
            for _ in range(a.reps):
                T.naive_convolve(l4, r4)
            torch.cuda.synchronize()
            print(name, "ok", flush=True)
            continue
        if name in ("EVVIEW255", "EVVIEW256"):   # EV of a view window (TMA tensor tiles)
            base_ = torch.rand((264,) * 3, dtype=torch.float64, device=dev)
            st_, sh_ = ((5,) * 3, (255,) * 3) if name == "EVVIEW255" else ((8,) * 3, (256,) * 3)
            v_ = T.View(base_, st_, sh_)
            o_ = torch.empty(3, dtype=torch.float64, device=dev)
            for _ in range(a.reps):
                T.expected_value_view(v_, out=o_)
            torch.cuda.synchronize()
            print(name, "ok", flush=True)
            continue
        if name in ("EV7", "EVF32"):   # expected value over odd innermost extents
            sh, dt = ((7,) * 9, torch.float64) if name == "EV7" else ((3000, 3000, 7), torch.float32)
            p_ = torch.rand(sh, dtype=dt, device=dev)
            o_ = torch.empty(len(sh), dtype=torch.float64, device=dev)
            for _ in range(a.reps):
                T.expected_value(p_, out=o_)
            torch.cuda.synchronize()
            print(name, "ok", flush=True)
            continue
        if name in ("ROWS7", "ROWS33", "ROWSB63"):   # short odd rows (row-window kernels)
            if name == "ROWSB63":
                a_ = torch.rand((2000, 2000, 63), device=dev)
                b_ = torch.rand((2001, 2000, 64), device=dev)
                c_ = torch.empty((2000, 2000, 63), device=dev)
                fn = lambda: T.apply_binary(a_, b_, "mul", out=c_, iter_shape=(2000, 2000, 63))
            else:
                sh = ((3000, 3000, 7), (2900, 2900, 5)) if name == "ROWS7" else \
                    ((3000, 1000, 33), (2900, 1000, 31))
                src_ = torch.rand(sh[1], device=dev)
                dst_ = torch.empty(sh[0], device=dev)
                fn = lambda: T.embed(dst_, src_)
            for _ in range(a.reps):
                fn()
            torch.cuda.synchronize()
            print(name, "ok", flush=True)
            continue
        if name in ("B2", "B3"):
            from triot_inputs import make_paper_inputs
            pin = make_paper_inputs(name)
            if name == "B2":
                x = torch.from_numpy(pin["a"]).to(dev)
                y = torch.from_numpy(pin["b"]).to(dev)
                fn = lambda: T.inner_product(x, y)
            else:
                x = torch.from_numpy(pin["x"]).to(dev)
                y = torch.from_numpy(pin["y"]).to(dev)
                z = torch.from_numpy(pin["z"]).to(dev)
                fn = lambda: T.fused_update(x, y, z)
            for _ in range(a.reps):
                fn()
            torch.cuda.synchronize()
            print(name, "ok", flush=True)
            continue
        inp = make_inputs(name)
        if name in ("C1", "C2", "C5"):
            src = torch.from_numpy(inp["src"]).to(dev)
            dst = torch.empty(inp["dst_shape"], dtype=src.dtype, device=dev)
            fn = lambda: T.embed(dst, src)
        elif name == "C3":
            p = torch.from_numpy(inp["p"]).to(dev)
            out = torch.empty(p.dim(), dtype=torch.float64, device=dev)
            fn = lambda: T.expected_value(p, out=out)
        else:
            x = torch.from_numpy(inp["a"]).to(dev)
            y = torch.from_numpy(inp["b"]).to(dev)
            c = torch.empty(inp["iter_shape"], dtype=torch.float64, device=dev)
            fn = lambda: T.apply_binary(x, y, "mul", out=c)
        for _ in range(a.reps):
            fn()
        torch.cuda.synchronize()
        print(name, "ok", flush=True)


if __name__ == "__main__":
    main()
