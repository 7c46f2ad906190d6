"""Per-call host cost of the Python API on a tiny op (C1), vs a one-element torch fill."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1608_00099_b200 as T
from triot_inputs import make_inputs
inp = make_inputs("C1")
src = torch.from_numpy(inp["src"]).cuda()
dst = torch.empty(inp["dst_shape"], dtype=torch.float64, device="cuda")
x = torch.empty(1, device="cuda")
for name, fn in (("embed C1", lambda: T.embed(dst, src)), ("torch fill 1 elem", lambda: x.fill_(1.0))):
    for _ in range(200): fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5000): fn()
    torch.cuda.synchronize()
    print(name, round((time.perf_counter() - t) / 5000 * 1e6, 2), "us/call")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    T.embed(dst, src)
s.synchronize()
print("side stream ok")
