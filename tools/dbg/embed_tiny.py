"""High-dimension tiny-extent embeds / products (isolated launches after an L2 scrub, GB/s)."""
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
cases = [((4,) * 14, (3,) * 14), ((7,) * 10, (5,) * 10), ((5,) * 12, (4,) * 12), ((3,) * 16, (2,) * 16), ((6,) * 10, (5,) * 10),
         ((8,) * 9, (5,) * 9), ((4,) * 14, (2,) * 14), ((9,) * 9, (8,) * 9), ((12,) * 8, (9,) * 8), ((16,) * 7, (11,) * 7)]
for dsh, ssh in cases:
    for dt in (torch.float32,):
        src = torch.rand(ssh, dtype=dt, device=DEV); dst = torch.empty(dsh, dtype=dt, device=DEV)
        nb = (src.numel() + dst.numel()) * src.element_size()
        desc = T.triot_plan_describe(0, [dsh, ssh], None, len(dsh), T._lib.TRIOT_F32, 0, (0, 0, 0))
        ms = timed(lambda: T.embed(dst, src))
        print(json.dumps({"op": "embed f32", "dst": f"({dsh[0]})^{len(dsh)}", "src": f"({ssh[0]})^{len(ssh)}", "MB": round(nb / 1e6), "plan": {k: desc.get(k) for k in ("D", "V", "R", "flat", "rows", "zmask")},
                          "us": round(ms * 1000, 1), "gbs": round(nb / ms / 1e6)}), flush=True)
        del src, dst
for ash, bsh in [((7,) * 10, (5,) * 10), ((6,) * 10, (5,) * 10), ((9,) * 9, (8,) * 9), ((5,) * 12, (4,) * 12)]:
    a = torch.rand(ash, dtype=torch.float32, device=DEV); b = torch.rand(bsh, dtype=torch.float32, device=DEV)
    it = tuple(min(x, y) for x, y in zip(ash, bsh)); c = torch.empty(it, dtype=torch.float32, device=DEV)
    nb = c.numel() * 4 * 3
    desc = T.triot_plan_describe(1, [None, ash, bsh], it, len(ash), T._lib.TRIOT_F32, T._lib.TRIOT_MUL, (0, 0, 0))
    ms = timed(lambda: T.apply_binary(a, b, "mul", out=c))
    print(json.dumps({"op": "mul f32", "a": f"({ash[0]})^{len(ash)}", "b": f"({bsh[0]})^{len(bsh)}", "MB": round(nb / 1e6), "plan": {k: desc.get(k) for k in ("D", "V", "R", "flat", "rows")},
                      "us": round(ms * 1000, 1), "gbs": round(nb / ms / 1e6)}), flush=True)
