"""Zero-padded embed and different-shape product across sizes, back to back in a CUDA graph
(steady state, us per op and effective GB/s), next to the torch idiom a user would write
instead (dst.zero_() + slice assignment; a[:m] * b[:m] into out) -- context, not a baseline arm.

    python tools/size_sweep.py > gpurun_out/size_sweep.jsonl
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1608_00099_b200 as T  # noqa: E402

DEV = torch.device("cuda:0")


def graph_us(fn, n=20, reps=3):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n):
            fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1000 / n)
    return best


def main():
    for n in (16, 32, 64, 96, 128, 192, 256, 384, 512):
        s = 3 * n // 4
        src = torch.randn((s, s, s), device=DEV)
        dst = torch.empty((n, n, n), device=DEV)
        nbytes = (src.numel() + dst.numel()) * 4

        def torch_embed():
            dst.zero_()
            dst[:s, :s, :s] = src

        t_us = graph_us(lambda: T.embed(dst, src))
        ref = dst.clone()
        r_us = graph_us(torch_embed)
        assert torch.equal(ref, dst)
        print(json.dumps({"op": "embed f32", "dst": [n] * 3, "src": [s] * 3, "bytes": nbytes,
                          "triot_us": round(t_us, 2), "triot_gbs": round(nbytes / t_us / 1e3, 1),
                          "torch_zero_plus_slice_us": round(r_us, 2),
                          "ratio": round(r_us / t_us, 2)}), flush=True)
    for n in (8, 16, 24, 32, 48, 64, 96, 128):
        a = torch.rand((n, n + n // 2, n), dtype=torch.float64, device=DEV)
        b = torch.rand((n + n // 4, n, n), dtype=torch.float64, device=DEV)
        out = torch.empty((n, n, n), dtype=torch.float64, device=DEV)
        nbytes = out.numel() * 8 * 3

        def torch_mul():
            torch.mul(a[:n, :n, :n], b[:n, :n, :n], out=out)

        t_us = graph_us(lambda: T.apply_binary(a, b, "mul", out=out))
        ref = out.clone()
        r_us = graph_us(torch_mul)
        assert torch.equal(ref, out)
        print(json.dumps({"op": "mul f64", "iter": [n] * 3, "bytes": nbytes,
                          "triot_us": round(t_us, 2), "triot_gbs": round(nbytes / t_us / 1e3, 1),
                          "torch_sliced_mul_us": round(r_us, 2),
                          "ratio": round(r_us / t_us, 2)}), flush=True)
    for d, n in ((6, 8), (6, 12), (6, 16), (4, 64), (4, 128), (3, 512)):
        p = torch.rand((n,) * d, dtype=torch.float64, device=DEV)
        p /= p.sum()
        m = torch.empty(d, dtype=torch.float64, device=DEV)
        nbytes = p.numel() * 8
        idx = [torch.arange(n, dtype=torch.float64, device=DEV).view([n if j == k else 1 for j in range(d)])
               for k in range(d)]

        def torch_ev():   # d weighted reductions over p
            for k in range(d):
                m[k] = (p * idx[k]).sum()

        t_us = graph_us(lambda: T.expected_value(p, out=m))
        got = m.clone()
        r_us = graph_us(torch_ev)
        assert torch.allclose(got, m, rtol=1e-10)
        print(json.dumps({"op": "expected value f64", "shape": [n] * d, "bytes": nbytes,
                          "triot_us": round(t_us, 2), "triot_gbs": round(nbytes / t_us / 1e3, 1),
                          "torch_d_weighted_sums_us": round(r_us, 2),
                          "ratio": round(r_us / t_us, 2)}), flush=True)


if __name__ == "__main__":
    main()
