"""Dense expected values whose rows take 16-byte vectors (isolated launches after an L2 scrub)."""
import json, os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1608_00099_b200 as T
DEV = torch.device("cuda:0")
scratch = torch.empty(512 << 20, dtype=torch.uint8, device=DEV)
clean = torch.ones(512 << 18, dtype=torch.int32, device=DEV)
for dt, ns in ((torch.float32, (2, 4, 12, 20, 28, 36, 60)), (torch.float64, (2, 6, 10, 14, 30, 34, 62))):
    for n in ns:
        esz = 4 if dt == torch.float32 else 8
        r = int(((256 << 20) // (n * esz)) ** 0.5) // 2 * 2
        p = torch.rand((r, r, n), dtype=dt, device=DEV)
        m = torch.empty(3, dtype=torch.float64, device=DEV)
        desc = T.triot_plan_describe(2, [tuple(p.shape)], None, 3, T._lib.TRIOT_F64 if esz == 8 else T._lib.TRIOT_F32, 0, (0, 0, 0))
        T.expected_value(p, out=m)
        ts = []
        for _ in range(7):
            scratch.fill_(1); clean.sum()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); T.expected_value(p, out=m); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ts.sort()
        nb = p.numel() * esz
        print(json.dumps({"dtype": str(dt)[6:], "n": n, "MB": round(nb / 1e6), "V": desc.get("V"), "R": desc.get("R"), "evrows": desc.get("evrows"),
                          "us": round(ts[3] * 1000, 1), "gbs": round(nb / ts[3] / 1e6)}), flush=True)
