"""Benchmark 4: per-call event time back to back, in a CUDA graph, and the kernel list."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1608_00099_b200 as T
dev = torch.device("cuda:0")
rng4 = np.random.default_rng(17)
l4 = torch.from_numpy(rng4.random((256, 8))).to(dev)
r4 = torch.from_numpy(rng4.random((256, 8))).to(dev)
o4 = torch.empty((511, 15), dtype=torch.float64, device=dev)
for _ in range(5): T.naive_convolve(l4, r4, out=o4)
torch.cuda.synchronize()
ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ea.record()
for _ in range(200): T.naive_convolve(l4, r4, out=o4)
eb.record(); torch.cuda.synchronize()
print("back to back us/call", ea.elapsed_time(eb) * 1000 / 200)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for _ in range(50): T.naive_convolve(l4, r4, out=o4)
g.replay(); torch.cuda.synchronize()
ea.record(); g.replay(); eb.record(); torch.cuda.synchronize()
print("graph us/call", ea.elapsed_time(eb) * 1000 / 50)
import time
t = time.perf_counter()
for _ in range(200): T.naive_convolve(l4, r4, out=o4)
torch.cuda.synchronize()
print("wall us/call", (time.perf_counter() - t) * 1e6 / 200)

# single warm launch
torch.cuda.synchronize()
ts = []
for _ in range(20):
    ea.record(); T.naive_convolve(l4, r4, out=o4); eb.record(); torch.cuda.synchronize()
    ts.append(ea.elapsed_time(eb) * 1000)
print("single launch us (min/median)", min(ts), sorted(ts)[10])
