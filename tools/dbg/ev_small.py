import json, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1608_00099_b200 as T
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tools"))
from size_sweep import graph_us
DEV = torch.device("cuda:0")
for shape in [(16,), (64,), (32, 32), (4,) * 6, (64, 64), (128, 64), (128, 128), (4,) * 7, (256, 128), (16,) * 4, (6,) * 6, (128, 128, 16), (8,) * 6, (10,) * 6]:
    p = torch.rand(shape, dtype=torch.float64, device=DEV); p /= p.sum()
    m = torch.empty(len(shape), dtype=torch.float64, device=DEV)
    desc = T.triot_plan_describe(2, [shape], None, len(shape), T._lib.TRIOT_F64, 0, (0, 0, 0))
    us = graph_us(lambda: T.expected_value(p, out=m), n=50)
    s1 = torch.empty((), dtype=torch.float64, device=DEV)
    pf = p.view(-1)
    tus = graph_us(lambda: torch.sum(pf, dim=(0,), out=s1), n=50)
    print(json.dumps({"shape": list(shape), "bytes": p.numel() * 8, "nsteps": desc.get("nsteps"), "ev_us": round(us, 2), "torch_sum_us": round(tus, 2)}), flush=True)
