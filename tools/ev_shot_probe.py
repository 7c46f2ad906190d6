"""One-shot expected-value kernel variants on C3 (diagnostic; builds tools/libevshot.so).

    python tools/ev_shot_probe.py [--ncu]     (--ncu: 3 launches per variant, no timing)

Per variant and grid cap: correctness against the library's result (rel 1e-12), one launch after
an L2 scrub (CUDA events, median of 9) and 20 back-to-back launches; a bare 134 MB read
(tools/membench) is timed the same way as the ceiling."""
import ctypes
import json
import os
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
TAIL = os.environ.get("EV_TAIL", "0")
SO = os.path.join(HERE, f"libevshot{TAIL}.so")


def build():
    srcs = [os.path.join(HERE, "ev_shot_probe.cu"),
            os.path.join(ROOT, "paper_1608_00099_b200", "csrc", "plan.cpp")]
    deps = srcs + [os.path.join(ROOT, "paper_1608_00099_b200", "csrc", f)
                   for f in ("kernels.cuh", "desc.h", "plan.hpp")]
    if not os.path.exists(SO) or any(os.path.getmtime(x) > os.path.getmtime(SO) for x in deps):
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                        "-lineinfo", f"-DTRIOT_EV_TAIL={TAIL}", "-shared", "-Xcompiler", "-fPIC", "-I",
                        os.path.join(ROOT, "include"), "-o", SO, *srcs], check=True)
    L = ctypes.CDLL(SO)
    L.probe_shot_c3.restype = ctypes.c_int
    L.probe_shot_c3.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
    L.probe_dyn_c3.restype = ctypes.c_int
    L.probe_dyn_c3.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 3 + [ctypes.c_void_p]
    L.probe_fx_c3.restype = ctypes.c_int
    L.probe_fx_c3.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 2 + [ctypes.c_void_p]
    L.probe_evk_c3.restype = ctypes.c_int
    L.probe_evk_c3.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] + [ctypes.c_void_p]
    L.probe_fx_info.restype = ctypes.c_int
    L.probe_fx_info.argtypes = [ctypes.c_int] + [ctypes.POINTER(ctypes.c_int)] * 3
    L.probe_dyn_info.restype = ctypes.c_int
    L.probe_dyn_info.argtypes = [ctypes.c_int] + [ctypes.POINTER(ctypes.c_int)] * 3
    L.probe_variant_info.restype = ctypes.c_int
    L.probe_variant_info.argtypes = [ctypes.c_int] + [ctypes.POINTER(ctypes.c_int)] * 3
    return L


def main():
    L = build()
    import paper_1608_00099_b200 as T
    from triot_inputs import make_inputs
    dev = torch.device("cuda:0")
    p = torch.from_numpy(make_inputs("C3")["p"]).to(dev)
    ref = T.expected_value(p).cpu()
    means = torch.zeros(6, dtype=torch.float64, device=dev)
    ws = torch.zeros(16 << 20, dtype=torch.uint8, device=dev)
    scratch = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    clean = torch.ones(512 << 18, dtype=torch.int32, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    ncu = "--ncu" in sys.argv
    caps = [0, sms * 8, sms * 16]
    configs = []
    if os.environ.get("EV_DYN"):
        for v in range(L.probe_dyn_variants()):
            j, bb, rg = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
            loc = L.probe_dyn_info(v, ctypes.byref(j), ctypes.byref(bb), ctypes.byref(rg))
            for rf in (0, 2, 4):
                for cap in (0, 2 * sms):
                    configs.append(({"kind": "dyn", "variant": v, "J": j.value, "B": bb.value,
                                     "regs": rg.value, "local": loc, "rforce": rf, "cap": cap},
                                    lambda v=v, rf=rf, cap=cap: L.probe_dyn_c3(
                                        p.data_ptr(), means.data_ptr(), ws.data_ptr(), v, rf, cap, s)))
    if os.environ.get("EV_FX"):
        for v in range(L.probe_fx_variants()):
            k_, rg, oc = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
            loc = L.probe_fx_info(v, ctypes.byref(k_), ctypes.byref(rg), ctypes.byref(oc))
            for bpsm in sorted({1, 2, oc.value}):
                if bpsm > oc.value:
                    continue
                configs.append(({"kind": "fx", "variant": v, "K": k_.value, "regs": rg.value,
                                 "local": loc, "occ": oc.value, "bpsm": bpsm},
                                lambda v=v, bpsm=bpsm: L.probe_fx_c3(
                                    p.data_ptr(), means.data_ptr(), ws.data_ptr(), v, bpsm, s) * 100000))
    if os.environ.get("EV_K"):
        for bpsm in (4, 6, 8, 12, 16):
            configs.append(({"kind": "evk", "bpsm": bpsm},
                            lambda bpsm=bpsm: L.probe_evk_c3(p.data_ptr(), means.data_ptr(),
                                                             ws.data_ptr(), bpsm, s) * 100000))
    for rec, fn in configs:
        means.zero_()
        r0 = fn()
        torch.cuda.synchronize()
        got = means.cpu()
        rec["grid"], rec["units"] = r0 // 100000, r0 % 100000
        rec["ok"] = bool(((got - ref).abs() <= 1e-12 * ref.abs()).all()) if TAIL == "0" else None
        rec["tail"] = int(TAIL)
        fn()
        torch.cuda.synchronize()
        rec["det"] = bool((means.cpu() == got).all())
        if ncu:
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            print(json.dumps(rec), flush=True)
            continue
        singles = []
        for _ in range(9):
            scratch.fill_(1)
            clean.sum()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            singles.append(a.elapsed_time(b) * 1000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            fn()
        b.record()
        torch.cuda.synchronize()
        singles.sort()
        rec.update(single_us=round(singles[4], 2), b2b_us=round(a.elapsed_time(b) * 1000 / 20, 2))
        print(json.dumps(rec), flush=True)
    if os.environ.get("EV_DYN") or os.environ.get("EV_FX") or os.environ.get("EV_K"):
        return
    nv = L.probe_variants()
    only = [int(x) for x in os.environ.get("EV_VARIANTS", "").split(",") if x]
    for v in range(nv):
        if only and v not in only:
            continue
        j, mb, rg = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        occ = L.probe_variant_info(v, ctypes.byref(j), ctypes.byref(mb), ctypes.byref(rg))
        for cap in caps:
            fn = lambda: L.probe_shot_c3(p.data_ptr(), means.data_ptr(), ws.data_ptr(), v, cap, s)
            grid = fn()
            torch.cuda.synchronize()
            got = means.cpu()
            ok = bool(((got - ref).abs() <= 1e-12 * ref.abs()).all()) if TAIL == "0" else None
            rec = {"tail": int(TAIL), "variant": v, "J": j.value, "minb": mb.value, "regs": rg.value, "occ": occ,
                   "cap": cap, "grid": grid, "ok": ok}
            if ncu:
                for _ in range(3):
                    fn()
                torch.cuda.synchronize()
                print(json.dumps(rec), flush=True)
                continue
            singles = []
            for _ in range(9):
                scratch.fill_(1)
                clean.sum()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                fn()
                b.record()
                torch.cuda.synchronize()
                singles.append(a.elapsed_time(b) * 1000)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                fn()
            b.record()
            torch.cuda.synchronize()
            singles.sort()
            rec.update(single_us=round(singles[4], 2), b2b_us=round(a.elapsed_time(b) * 1000 / 20, 2))
            print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
