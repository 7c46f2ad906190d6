"""Aligned expected values, f32 vs f64, large (ncu-free, isolated launches after an L2 scrub)."""
import json, os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1608_00099_b200 as T
DEV = torch.device("cuda:0")
scratch = torch.empty(512 << 20, dtype=torch.uint8, device=DEV)
clean = torch.ones(512 << 18, dtype=torch.int32, device=DEV)
for dt, sh in ((torch.float32, (512, 512, 512)), (torch.float64, (512, 512, 256)), (torch.float32, (32,) * 5 + (16,)),
               (torch.float32, (1024, 1024, 1024)), (torch.float64, (1024, 1024, 512)), (torch.float32, (4096, 4096, 4)),
               (torch.float32, (4096, 4096, 12)), (torch.float64, (4096, 4096, 6))):
    p = torch.rand(sh, dtype=dt, device=DEV)
    m = torch.empty(len(sh), dtype=torch.float64, device=DEV)
    T.expected_value(p, out=m)
    ts = []
    for _ in range(7):
        scratch.fill_(1); clean.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); T.expected_value(p, out=m); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    nb = p.numel() * p.element_size()
    print(json.dumps({"dtype": str(dt)[6:], "shape": list(sh), "MB": round(nb / 1e6), "us": round(ts[3] * 1000, 1), "gbs": round(nb / ts[3] / 1e6)}), flush=True)
    del p
