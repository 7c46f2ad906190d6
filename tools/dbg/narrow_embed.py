"""Embeds / products whose rows only admit 16-byte vectors (isolated launches, GB/s)."""
import json, os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1608_00099_b200 as T
DEV = torch.device("cuda:0")
scratch = torch.empty(512 << 20, dtype=torch.uint8, device=DEV)
clean = torch.ones(512 << 18, dtype=torch.int32, device=DEV)
def timed(fn):
    fn(); ts = []
    for _ in range(7):
        scratch.fill_(1); clean.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ts.sort(); return ts[3]
for dt, esz, ns in ((torch.float32, 4, (12, 20, 28)), (torch.float64, 8, (6, 10, 14, 30))):
    for n in ns:
        r = int(((384 << 20) // (n * esz)) ** 0.5)
        dst = torch.empty((r, r, n), dtype=dt, device=DEV)
        src = torch.rand((r - 100, r - 100, n - (4 if esz == 4 else 2)), dtype=dt, device=DEV)
        nb = (src.numel() + dst.numel()) * esz
        code = T._lib.TRIOT_F32 if esz == 4 else T._lib.TRIOT_F64
        desc = T.triot_plan_describe(0, [tuple(dst.shape), tuple(src.shape)], None, 3, code, 0, (0, 0, 0))
        ms = timed(lambda: T.embed(dst, src))
        print(json.dumps({"op": "embed", "dtype": str(dt)[6:], "n": n, "m": src.shape[-1], "MB": round(nb / 1e6), "V": desc.get("V"), "rows": desc.get("rows"),
                          "us": round(ms * 1000, 1), "gbs": round(nb / ms / 1e6)}), flush=True)
        a = torch.rand((r, r, n), dtype=dt, device=DEV); b = torch.rand((r, r + 1, n + (4 if esz == 4 else 2)), dtype=dt, device=DEV)
        c = dst
        nb = 3 * c.numel() * esz
        desc = T.triot_plan_describe(1, [None, tuple(a.shape), tuple(b.shape)], tuple(c.shape), 3, code, T._lib.TRIOT_MUL, (0, 0, 0))
        ms = timed(lambda: T.apply_binary(a, b, "mul", out=c))
        print(json.dumps({"op": "mul", "dtype": str(dt)[6:], "n": n, "MB": round(nb / 1e6), "V": desc.get("V"), "rows": desc.get("rows"),
                          "us": round(ms * 1000, 1), "gbs": round(nb / ms / 1e6)}), flush=True)
        del a, b, src, dst, c
