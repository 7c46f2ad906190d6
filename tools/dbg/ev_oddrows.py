"""Dense expected values with odd innermost extents (isolated launches after an L2 scrub, GB/s)."""
import json, os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1608_00099_b200 as T
DEV = torch.device("cuda:0")
scratch = torch.empty(512 << 20, dtype=torch.uint8, device=DEV)
clean = torch.ones(512 << 18, dtype=torch.int32, device=DEV)
for dt in (torch.float64, torch.float32):
    for n in (tuple(int(x) for x in os.environ["EVODD_N"].split(",")) if os.environ.get("EVODD_N") else (7, 31, 33, 45, 63, 65, 127, 255, 999)):
        rows = (256 << 20) // (n * (8 if dt == torch.float64 else 4))
        r = int(rows ** 0.5)
        p = torch.rand((r, r, n), dtype=dt, device=DEV)
        m = torch.empty(3, dtype=torch.float64, device=DEV)
        desc = T.triot_plan_describe(2, [tuple(p.shape)], None, 3, T._lib.TRIOT_F64 if dt == torch.float64 else T._lib.TRIOT_F32, 0, (0, 0, 0))
        T.expected_value(p, out=m)
        ts = []
        for _ in range(7):
            scratch.fill_(1); clean.sum()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); T.expected_value(p, out=m); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ts.sort()
        nb = p.numel() * p.element_size()
        print(json.dumps({"dtype": str(dt)[6:], "shape": list(p.shape), "MB": round(nb / 1e6), "flat": desc.get("flat"), "evrows": desc.get("evrows"), "V": desc.get("V"),
                          "us": round(ts[3] * 1000, 1), "gbs": round(nb / ts[3] / 1e6, 0)}), flush=True)
