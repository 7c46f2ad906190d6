"""Per-block timeline of the EV kernel on C3: bulk-copy kernel, or the default LDG kernel with
--ldg (diagnostic; builds tools/libevprobe.so)."""
import ctypes
import json
import os
import subprocess
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
DEFS = os.environ.get("EVPROBE_DEFS", "").split()   # e.g. "-DTRIOT_EV_LL=0": A/B of the tail
SO = os.path.join(HERE, "libevprobe%s.so" % ("_" + "".join(c for c in "".join(DEFS) if c.isalnum()) if DEFS else ""))


def build():
    srcs = [os.path.join(HERE, "ev_probe.cu"),
            os.path.join(ROOT, "paper_1608_00099_b200", "csrc", "plan.cpp")]
    if not os.path.exists(SO) or any(os.path.getmtime(x) > os.path.getmtime(SO) for x in srcs):
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                        "-shared", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"), *DEFS,
                        "-o", SO, *srcs], check=True)
    L = ctypes.CDLL(SO)
    for f in (L.probe_ev_c3, L.probe_ev_ldg_c3):
        f.restype = ctypes.c_int
        f.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int, ctypes.c_void_p]
    L.probe_dot_b2.restype = ctypes.c_int
    L.probe_dot_b2.argtypes = [ctypes.c_void_p] * 5 + [ctypes.c_int, ctypes.c_void_p]
    return L


def main():
    L = build()
    from triot_inputs import make_inputs
    dev = torch.device("cuda:0")
    p = torch.from_numpy(make_inputs("C3")["p"]).to(dev)
    means = torch.zeros(6, dtype=torch.float64, device=dev)
    ws = torch.zeros(1 << 20, dtype=torch.uint8, device=dev)
    trace = torch.zeros(4096 * 8, dtype=torch.int64, device=dev)
    scratch = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    clean = torch.ones(512 << 18, dtype=torch.int32, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    ldg = "--ldg" in sys.argv or "--dot" in sys.argv
    probe = L.probe_ev_ldg_c3 if ldg else L.probe_ev_c3
    nblk = sms * (4 if ldg else 1)
    if "--dot" in sys.argv:
        from triot_inputs import make_paper_inputs
        inp = make_paper_inputs("B2")
        A = torch.from_numpy(inp["a"]).to(dev)
        B = torch.from_numpy(inp["b"]).to(dev)
        probe = lambda p_, m_, w_, t_, n_, s_: L.probe_dot_b2(A.data_ptr(), B.data_ptr(), m_, w_,
                                                               t_, n_, s_)
    dump = []
    nrep = 3
    if "--dump" in sys.argv:   # per-block traces of many launches (per-SM statistics offline)
        nrep = int(sys.argv[sys.argv.index("--dump") + 1])
    for rep in range(nrep):
        scratch.fill_(1)
        clean.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        grid = probe(p.data_ptr(), means.data_ptr(), ws.data_ptr(), trace.data_ptr(), nblk, s)
        b.record()
        torch.cuda.synchronize()
        assert grid > 0, grid
        tr = trace[: grid * 8].view(grid, 8).cpu().numpy().astype(np.int64)
        t0 = tr[:, 0].min()
        if "--dump" in sys.argv:
            dump.append(np.concatenate([tr[:, :7] - t0, tr[:, 7:8]], axis=1).astype(np.int32))
            continue
        rel = (tr[:, :5] - t0) / 1000.0
        pct = lambda col, qs: [round(float(np.percentile(rel[:, col], q)), 2) for q in qs]
        print(json.dumps({
            "grid": grid, "event_us": round(a.elapsed_time(b) * 1000, 2),
            "start_us": pct(0, (0, 50, 100)),
            "first_stage_us": pct(1, (0, 50, 100)),
            "loop_end_us": pct(2, (0, 10, 50, 90, 100)),
            "ticket_us": pct(3, (0, 50, 100)),
            "exit_last_us": round(float(rel[:, 4].max()), 2),
            "last_block_loads_done_us": round(float(((tr[:, 5].max()) - t0) / 1000.0), 2),
            "last_block_reduced_us": round(float(((tr[:, 6].max()) - t0) / 1000.0), 2),
            "slowest_blocks_sm": [int(x) for x in tr[np.argsort(-tr[:, 2])[:8], 7]],
            "fastest_blocks_sm": [int(x) for x in tr[np.argsort(tr[:, 2])[:8], 7]],
            "means": means.cpu().tolist()}), flush=True)
    if dump:
        out = os.path.join(ROOT, "gpurun_out", "ev_trace_dump.npy")
        np.save(out, np.stack(dump))
        print("saved", out, np.stack(dump).shape)


if __name__ == "__main__":
    main()
