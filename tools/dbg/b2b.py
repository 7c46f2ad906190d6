"""Back-to-back calls of each paper benchmark and config op in a CUDA graph (us per call)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1608_00099_b200 as T
from triot_inputs import make_inputs, make_paper_inputs
dev = torch.device("cuda:0")
if os.environ.get("TRIOT_POLICY"):   # "mode,blocks_per_sm"
    T.triot_set_launch_policy(*(int(x) for x in os.environ["TRIOT_POLICY"].split(",")))
b1 = make_paper_inputs("B1"); y1 = torch.from_numpy(b1["src"]).to(dev)
x1 = torch.empty(b1["dst_shape"], dtype=torch.float64, device=dev)
b2 = make_paper_inputs("B2"); a2, bb2 = torch.from_numpy(b2["a"]).to(dev), torch.from_numpy(b2["b"]).to(dev)
o2 = torch.empty(1, dtype=torch.float64, device=dev)
b3 = make_paper_inputs("B3"); x3 = torch.from_numpy(b3["x"]).to(dev)
y3, z3 = torch.from_numpy(b3["y"]).to(dev), torch.from_numpy(b3["z"]).to(dev)
c3 = torch.from_numpy(make_inputs("C3")["p"]).to(dev); m3 = torch.empty(6, dtype=torch.float64, device=dev)
cases = {"B1": lambda: T.embed(x1, y1), "B2": lambda: T.inner_product(a2, bb2, out=o2),
         "B3": lambda: T.fused_update(x3, y3, z3), "C3": lambda: T.expected_value(c3, out=m3)}
out = {}
for n, fn in cases.items():
    for _ in range(3): fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(20): fn()
    g.replay(); torch.cuda.synchronize()
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(3):
        ea.record(); g.replay(); eb.record(); torch.cuda.synchronize()
        ts.append(ea.elapsed_time(eb) * 1000 / 20)
    out[n] = round(min(ts), 2)
print(json.dumps(out))
