"""Throughput of the general path on awkward shapes (diagnostic): odd / prime innermost extents
(narrow or scalar vector widths), high d, crops, misaligned bases.  One line per case:
effective GB/s (algorithmic bytes / single-launch time after a clean L2 scrub)."""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1608_00099_b200 as T  # noqa: E402

dev = torch.device("cuda:0")
if "--policy" in sys.argv:   # e.g. --policy 5,0: row windows off (flat vectors), A/B runs
    _m, _b = (int(x) for x in sys.argv[sys.argv.index("--policy") + 1].split(","))
    T.triot_set_launch_policy(_m, _b)
scratch = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
clean = torch.ones(512 << 18, dtype=torch.int32, device=dev)


def timed(fn, reps=5):
    fn()
    ts = []
    for _ in range(reps):
        scratch.fill_(1)
        clean.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


def embed_case(name, dst_shape, src_shape, dtype=torch.float32, off=0, soff=0):
    src = torch.rand(math.prod(src_shape) + soff, dtype=dtype, device=dev)[soff:].view(src_shape)
    n = math.prod(dst_shape)
    buf = torch.empty(n + off, dtype=dtype, device=dev)
    dst = buf[off:].view(dst_shape)
    ms = timed(lambda: T.embed(dst, src))
    esz = src.element_size()
    nbytes = (math.prod(min(a, b) for a, b in zip(src_shape, dst_shape)) + n) * esz
    d = len(dst_shape)
    plan = T.triot_plan_describe(0, [dst_shape, src_shape], None, d,
                                 0 if dtype == torch.float32 else 1, 0,
                                 (off * esz % 32, soff * esz % 32, 0))
    print(json.dumps({"case": name, "op": "embed", "us": round(ms * 1e3, 1),
                      "gbs": round(nbytes / ms / 1e6, 1), "V": plan["V"], "D": plan["D"],
                      "geom": "rows" if plan["rows"] else "flat" if plan["flat"] else "vec",
                      "vec": [t["vec"] for t in plan["t"]]}), flush=True)


def binary_case(name, a_shape, b_shape, dtype=torch.float64, aoff=0, coff=0):
    a = torch.rand(math.prod(a_shape) + aoff, dtype=dtype, device=dev)[aoff:].view(a_shape)
    b = torch.rand(b_shape, dtype=dtype, device=dev)
    ish = tuple(min(x, y) for x, y in zip(a_shape, b_shape))
    c = torch.empty(math.prod(ish) + coff, dtype=dtype, device=dev)[coff:].view(ish)
    ms = timed(lambda: T.apply_binary(a, b, "mul", out=c))
    nbytes = 3 * math.prod(ish) * a.element_size()
    d = len(ish)
    esz = a.element_size()
    plan = T.triot_plan_describe(1, [None, a_shape, b_shape], None, d,
                                 0 if dtype == torch.float32 else 1, 2,
                                 (coff * esz % 32, aoff * esz % 32, 0))
    print(json.dumps({"case": name, "op": "binary", "us": round(ms * 1e3, 1),
                      "gbs": round(nbytes / ms / 1e6, 1), "V": plan["V"], "D": plan["D"],
                      "geom": "rows" if plan["rows"] else "flat" if plan["flat"] else "vec",
                      "vec": [t["vec"] for t in plan["t"]]}), flush=True)


def ev_case(name, shape, dtype=torch.float64, off=0):
    n = math.prod(shape)
    buf = torch.rand(n + off, dtype=dtype, device=dev)
    p = buf[off:].view(shape)
    out = torch.empty(len(shape), dtype=torch.float64, device=dev)
    ms = timed(lambda: T.expected_value(p, out=out))
    nbytes = n * p.element_size()
    print(json.dumps({"case": name, "op": "ev", "us": round(ms * 1e3, 1),
                      "gbs": round(nbytes / ms / 1e6, 1)}), flush=True)


if "--rows" in sys.argv:   # short odd rows: row windows vs flat vectors (run with --policy 5,0)
    embed_case("rows: embed f32 (3000,3000,7) <- (2900,2900,5)", (3000, 3000, 7), (2900, 2900, 5))
    embed_case("rows: embed f32 (8192,4096,3) <- (8000,4000,3)", (8192, 4096, 3), (8000, 4000, 3))
    embed_case("rows: embed f64 (1000,1000,15) <- (1000,999,15)", (1000, 1000, 15), (1000, 999, 15),
               dtype=torch.float64)
    embed_case("rows: embed f32 (3000,1000,33) <- (2900,1000,31)", (3000, 1000, 33), (2900, 1000, 31))
    embed_case("rows: embed f32 (3000,3000,15) <- (2900,2900,13)", (3000, 3000, 15), (2900, 2900, 13))
    embed_case("rows: embed f32 (3000,1000,31) <- (2900,1000,29)", (3000, 1000, 31), (2900, 1000, 29))
    embed_case("rows: embed f64 (3000,3000,7) <- (2900,2900,5)", (3000, 3000, 7), (2900, 2900, 5),
               dtype=torch.float64)
    embed_case("rows: embed f32 (7)^8 <- (5)^8", (7,) * 8, (5,) * 8)
    embed_case("rows: embed f32 (5)^10 <- (4)^10", (5,) * 10, (4,) * 10)
    embed_case("rows: crop f32 (4096,512,3) <- (4100,600,7)", (4096, 512, 3), (4100, 600, 7))
    embed_case("rows: embed f32 (4096,4096,5) <- same, dst misaligned", (4096, 4096, 5),
               (4096, 4096, 5), off=1)
    embed_case("rows: C2 dst misaligned by 1 element", (512,) * 3, (384,) * 3, off=1)
    embed_case("rows: merged copy (4096,4096,5) <- same, dst misaligned", (4096, 4096, 5),
               (4096, 4096, 5), off=1)
    embed_case("rows: merged pad (512)^3 <- (500,512,512), dst misaligned", (512,) * 3,
               (500, 512, 512), off=1)
    embed_case("rows: C2 src misaligned by 1 element", (512,) * 3, (384,) * 3, soff=1)
    embed_case("rows: f64 pad (128)^4 from (100)^4, dst misaligned", (128,) * 4, (100,) * 4,
               dtype=torch.float64, off=1)
    binary_case("rows: binary f64 (64)^4 vs (80)^4, c misaligned", (64,) * 4, (80,) * 4, coff=1)
    binary_case("rows: binary f64 (64)^4 vs (80)^4, a misaligned", (64,) * 4, (80,) * 4, aoff=1)
    binary_case("rows: binary f64 (3000,3001,7) x (3001,3000,7)", (3000, 3001, 7), (3001, 3000, 7))
    binary_case("rows: binary f32 (4000,4001,3) x (4001,4000,3)", (4000, 4001, 3), (4001, 4000, 3),
                dtype=torch.float32)
    binary_case("rows: binary f64 (200,300,401,5) x (201,300,400,5)", (200, 300, 401, 5),
                (201, 300, 400, 5))
    binary_case("rows: binary f32 (2000,2000,63) x (2001,2000,64)", (2000, 2000, 63),
                (2001, 2000, 64), dtype=torch.float32)
    sys.exit(0)
if "--views" in sys.argv:   # NEXT-1 views: windows at aligned and odd offsets
    def view_ev(name, base_shape, start, shape, dtype=torch.float64):
        base = torch.rand(base_shape, dtype=dtype, device=dev)
        v = T.View(base, start, shape)
        out = torch.empty(len(shape), dtype=torch.float64, device=dev)
        ms = timed(lambda: T.expected_value_view(v, out=out))
        nbytes = math.prod(shape) * base.element_size()
        print(json.dumps({"case": name, "op": "ev_view", "us": round(ms * 1e3, 1),
                          "gbs": round(nbytes / ms / 1e6, 1)}), flush=True)

    def view_embed(name, dbase, dstart, sbase, sstart, shape, dtype=torch.float32):
        db = torch.zeros(dbase, dtype=dtype, device=dev)
        sb = torch.rand(sbase, dtype=dtype, device=dev)
        dv, sv = T.View(db, dstart, shape), T.View(sb, sstart, shape)
        ms = timed(lambda: T.embed_view(dv, sv))
        nbytes = 2 * math.prod(shape) * db.element_size()
        print(json.dumps({"case": name, "op": "embed_view", "us": round(ms * 1e3, 1),
                          "gbs": round(nbytes / ms / 1e6, 1)}), flush=True)

    view_ev("views: EV f64 (256)^3 window of (264)^3 at (8,8,8)", (264,) * 3, (8, 8, 8), (256,) * 3)
    view_ev("views: EV f64 (256)^3 window of (264)^3 at (5,5,5)", (264,) * 3, (5, 5, 5), (256,) * 3)
    view_ev("views: EV f64 (255)^3 window of (264)^3 at (5,5,5)", (264,) * 3, (5, 5, 5), (255,) * 3)
    view_ev("views: EV f32 (500)^3 window of (512)^3 at (3,3,3)", (512,) * 3, (3, 3, 3), (500,) * 3,
            dtype=torch.float32)
    view_embed("views: embed f32 (384)^3 into (512)^3 at (64,64,64)", (512,) * 3, (64,) * 3,
               (384,) * 3, (0,) * 3, (384,) * 3)
    view_embed("views: embed f32 (384)^3 into (512)^3 at (63,63,63)", (512,) * 3, (63,) * 3,
               (384,) * 3, (0,) * 3, (384,) * 3)
    view_embed("views: embed f32 window (383)^3 of (400)^3 at (1,1,1) into (512)^3 at (5,5,5)",
               (512,) * 3, (5,) * 3, (400,) * 3, (1,) * 3, (383,) * 3)
    sys.exit(0)
if "--evodd" in sys.argv:   # dense EV with odd innermost extents (row tiles vs --policy 5,0 flat)
    ev_case("evodd: EV f64 (7,)*9", (7,) * 9)
    ev_case("evodd: EV f32 (3000,3000,7)", (3000, 3000, 7), dtype=torch.float32)
    ev_case("evodd: EV f64 (3000,3000,7)", (3000, 3000, 7))
    ev_case("evodd: EV f32 (2000,2000,15)", (2000, 2000, 15), dtype=torch.float32)
    ev_case("evodd: EV f64 (1000,1000,31)", (1000, 1000, 31))
    ev_case("evodd: EV f32 (4000,4000,3)", (4000, 4000, 3), dtype=torch.float32)
    ev_case("evodd: EV f64 (5,)*11", (5,) * 11)
    sys.exit(0)
if "--big" in sys.argv:   # odd innermost extents at sizes past the launch-bound regime
    embed_case("big: embed f32 (3000,3000,7) <- (2900,2900,5)", (3000, 3000, 7), (2900, 2900, 5))
    embed_case("big: embed f32 (8192,4096,3) <- (8000,4000,3)", (8192, 4096, 3), (8000, 4000, 3))
    embed_case("big: embed f64 (1000,1000,15) <- (1000,999,15)", (1000, 1000, 15), (1000, 999, 15),
               dtype=torch.float64)
    binary_case("big: binary f64 (3000,3001,7) x (3001,3000,7)", (3000, 3001, 7), (3001, 3000, 7))
    binary_case("big: binary f32 (4000,4001,3) x (4001,4000,3)", (4000, 4001, 3), (4001, 4000, 3),
                dtype=torch.float32)
    ev_case("big: EV f64 (7,)*9", (7,) * 9)
    ev_case("big: EV f32 (3000,3000,7)", (3000, 3000, 7), dtype=torch.float32)
    sys.exit(0)
embed_case("pad 2-D, innermost 999 (odd: 1-element vectors)", (1000, 1001), (900, 999))
embed_case("pad 2-D, innermost 1000 (16-B vectors)", (1000, 1000), (900, 998))
embed_case("pad 2-D, innermost 1024", (1000, 1024), (900, 1000))
embed_case("crop 3-D to innermost 3", (4096, 512, 3), (4100, 600, 7))
embed_case("pad d=16 (2)^16 from (1,2,...)", (2,) * 16 + (), (1,) + (2,) * 15)
embed_case("pad d=8 (7)^8 from (5)^8 (prime)", (7,) * 8, (5,) * 8)
embed_case("pad d=10 (5)^10 from (4)^10", (5,) * 10, (4,) * 10)
embed_case("C2 with dst misaligned by 1 element", (512,) * 3, (384,) * 3, off=1)
embed_case("f64 pad (128)^4 from (100)^4", (128,) * 4, (100,) * 4, dtype=torch.float64)
binary_case("binary f64 innermost 5 (scalar)", (200, 300, 401, 5), (201, 300, 400, 5))
binary_case("binary f64 (64)^4 vs (80)^4", (64, 64, 64, 64), (80, 80, 80, 80))
binary_case("binary f32 d=12 (4)^12 vs (5)^12", (4,) * 12, (5,) * 12, dtype=torch.float32)
ev_case("EV f64 (4096, 4096)", (4096, 4096))
ev_case("EV f64 (7,)*9 (odd innermost: LDG path)", (7,) * 9)
ev_case("EV f32 (512,)*3", (512,) * 3, dtype=torch.float32)
ev_case("EV f64 C3 misaligned by 1 (LDG path)", (16,) * 6, off=1)
