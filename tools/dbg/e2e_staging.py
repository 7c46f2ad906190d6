"""e2e step time (all four legs on separate streams) vs the host-pipeline staging size."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1608_00099_b200 as T
from triot_inputs import make_inputs
dev = torch.device("cuda:0")
h = {n: make_inputs(n) for n in ("C2", "C3", "C4", "C5")}
src2 = torch.from_numpy(h["C2"]["src"]).pin_memory(); p3 = torch.from_numpy(h["C3"]["p"]).pin_memory()
a4 = torch.from_numpy(h["C4"]["a"]).pin_memory(); b4 = torch.from_numpy(h["C4"]["b"]).pin_memory()
src5 = torch.from_numpy(h["C5"]["src"]).pin_memory()
dst2 = torch.empty(h["C2"]["dst_shape"], dtype=torch.float32).pin_memory()
c4 = torch.empty(h["C4"]["iter_shape"], dtype=torch.float64).pin_memory()
dst5 = torch.empty(h["C5"]["dst_shape"], dtype=torch.float32).pin_memory()
m3 = torch.empty(6, dtype=torch.float64).pin_memory()
main_s = torch.cuda.current_stream(); side = [torch.cuda.Stream(dev) for _ in range(4)]
legs = [lambda: T.embed_host(dst2, src2, device=dev),
        lambda: m3.copy_(T.expected_value(p3.to(dev, non_blocking=True)), non_blocking=True),
        lambda: T.apply_binary_host(a4, b4, "mul", out=c4, device=dev),
        lambda: T.embed_host(dst5, src5, device=dev)]
def run():
    for i, f in enumerate(legs):
        side[i].wait_stream(main_s)
        with torch.cuda.stream(side[i]): f()
    for s in side: main_s.wait_stream(s)
for mb in (256, 512, 1024, 128, 256, 512):
    T.api.STAGING_BYTES = mb << 20; T.api._ws_cache.clear()
    run(); torch.cuda.synchronize()
    ts = []
    for _ in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(main_s); run(); b.record(main_s); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    print(json.dumps({"staging_MB": mb, "ms": [round(t, 2) for t in ts]}), flush=True)
