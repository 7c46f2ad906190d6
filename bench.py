"""bench.py -- effective HBM GB/s of the TRIOT hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one pass of the whole hot path over the BASELINE workloads that are bandwidth
measurements: C2 embed (f32, (384)^3 -> (512)^3), C3 expected value (f64, (16)^6),
C4 product (f64, A (32,48,24,40,36) x B (40,32,32,32,32) over (32,32,24,32,32)) and
C5 embed (f32, (3)^14 -> (4)^14), in that order on one stream.  C1 (75 KB, launch-bound) is
reported separately as latency.  value = algorithmic bytes (read + written)
of the K timed steps / device time; inputs are resident in HBM before the timed region; the
step moves 2.6 GB, ≫ the 126 MB L2, so each op's inputs were evicted by its predecessor
(no extra flush).  Device time = CUDA events on the launching stream, max over ranks.

N > 1 (torchrun): ONE global instance of each config is partitioned over the ranks along its
outermost loops (parallel.leading_box: axis-0 slabs, or axis-0 indices shared by rank
groups that split axis 1 when there are more ranks than indices -- C5's (4)^14 at 8 GPUs).
Embed and product need no collective; the expected value is each rank's triot_expected_value_
offset on its slab (global coordinates), an NCCL all_gather of the d doubles and triot_sum_rows
in rank order (deterministic).  Strong scaling: value = the global instance's bytes per step x K
/ max-over-ranks time.

--impl reference: the CPU oracle (oracle/, plain C, 1 thread) on a bounded slab of the same
workload per step (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from triot_inputs import CONFIGS, make_inputs  # noqa: E402

METRIC = "effective HBM GB/s and % of B200 peak per op (embed/binary/expected value)"
UNIT = "GB/s"
NOMINAL_HBM_GBS = 8000.0
WORKLOAD = "C2+C3+C4+C5"
STEP_OPS = ("C2", "C3", "C4", "C5")


def algorithmic_bytes(name: str) -> int:
    """Bytes read + written per op: embed reads the src elements inside dst
    and writes all of dst; binary reads a and b over iter and writes c; EV reads p and writes
    d doubles."""
    c = CONFIGS[name]
    esz = 4 if c.dtype == "f32" else 8
    sh = c.shapes
    if c.op == "embed":
        rd = math.prod(min(a, b) for a, b in zip(sh["src"], sh["dst"])) * esz
        wr = math.prod(sh["dst"]) * esz
    elif c.op == "ev":
        rd, wr = math.prod(sh["p"]) * esz, len(sh["p"]) * 8
    else:
        rd, wr = 2 * math.prod(sh["iter"]) * esz, math.prod(sh["iter"]) * esz
    return rd + wr


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi SM clocks + throttle reasons, sampled every 50 ms while running."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self.proc = None
        self.marks = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.samples.append((time.time(), parts))

    def mark(self):
        self.marks.append(time.time())

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        lo, hi = (self.marks[0], self.marks[-1]) if len(self.marks) >= 2 else (0, 1e30)
        inwin = [p for t, p in self.samples if lo - 0.06 <= t <= hi + 0.06]
        use = inwin if inwin else [p for _, p in self.samples]

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(p[1]) for p in use if num(p[1]) is not None]
        mx = [num(p[2]) for p in use if num(p[2]) is not None]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for p in use:
            for nm, v in zip(names, p[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(use),
                "window": "timed region" if inwin else "whole run"}


# ----------------------------------------------------------------------------- our arm

def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    # the partitioned (multi-GPU) path; --split-test runs it at world size 1 (a one-rank NCCL
    # group, the offset EV + all_gather + sum_rows) so a one-GPU box exercises every line of it
    split = world > 1 or args.split_test
    import paper_1608_00099_b200 as T

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    if split:
        if "MASTER_ADDR" not in os.environ:   # --split-test without torchrun: a one-rank group
            import socket
            so = socket.socket()
            so.bind(("127.0.0.1", 0))
            os.environ["MASTER_ADDR"] = "127.0.0.1"
            os.environ["MASTER_PORT"] = str(so.getsockname()[1])
            so.close()
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
        try:
            nv = ".".join(map(str, torch.cuda.nccl.version()))
        except Exception:
            nv = "?"
        print(f"[bench rank {rank}/{world}] NCCL process group up on {dev} "
              f"(backend {dist.get_backend()}, NCCL {nv})", file=sys.stderr, flush=True)

    # ---- inputs resident in HBM (init excluded from timing): this rank's box of each
    # config (the whole config at N = 1)
    host = {n: make_inputs(n) for n in ("C1",) + STEP_OPS}
    sl = slab_plan(host, world, rank)
    g = {}
    g["src2"] = torch.from_numpy(sl["C2"]["src"]).to(dev)
    g["dst2"] = torch.empty(sl["C2"]["dst_shape"], dtype=torch.float32, device=dev)
    g["p3"] = torch.from_numpy(sl["C3"]["p"]).to(dev)
    g["m3"] = torch.empty(6, dtype=torch.float64, device=dev)
    g["a4"] = torch.from_numpy(sl["C4"]["a"]).to(dev)
    g["b4"] = torch.from_numpy(sl["C4"]["b"]).to(dev)
    g["c4"] = torch.empty(sl["C4"]["iter_shape"], dtype=torch.float64, device=dev)
    g["src5"] = torch.from_numpy(sl["C5"]["src"]).to(dev)
    g["dst5"] = torch.empty(sl["C5"]["dst_shape"], dtype=torch.float32, device=dev)
    if split:
        g["g3"] = torch.empty(world * 6, dtype=torch.float64, device=dev)
        g["r3"] = torch.empty(6, dtype=torch.float64, device=dev)
    off3 = sl["C3"]["offset"]
    stream = torch.cuda.current_stream(dev)

    def ev_step():
        if not split:
            T.expected_value(g["p3"], out=g["m3"])
        else:  # the one exchange: d doubles per rank, summed in rank order
            T.expected_value(g["p3"], out=g["m3"], offset=off3)
            dist.all_gather_into_tensor(g["g3"], g["m3"])
            T.sum_rows(g["g3"].view(world, 6), out=g["r3"])

    def step(evs=None):
        T.embed(g["dst2"], g["src2"])
        if evs is not None:
            evs[0].record(stream)
        ev_step()
        if evs is not None:
            evs[1].record(stream)
        T.apply_binary(g["a4"], g["b4"], "mul", out=g["c4"], iter_shape=sl["C4"]["iter_shape"])
        if evs is not None:
            evs[2].record(stream)
        T.embed(g["dst5"], g["src5"])
        if evs is not None:
            evs[3].record(stream)

    sampler = ClockSampler(dev.index if dev.index is not None else 0)
    sampler.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    # ---- timed region: K steps, events between ops, barrier + sync on both sides
    K = args.steps
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K)]
    e_start = torch.cuda.Event(enable_timing=True)
    if split:
        dist.barrier()
    torch.cuda.synchronize(dev)
    sampler.mark()
    e_start.record(stream)
    for k in range(K):
        step(evs[k])
    torch.cuda.synchronize(dev)
    sampler.mark()
    if split:
        dist.barrier()
    total_ms = e_start.elapsed_time(evs[-1][3])
    per_op_ms = {n: 0.0 for n in STEP_OPS}
    for k in range(K):
        prev = e_start if k == 0 else evs[k - 1][3]
        marks = [prev] + evs[k]
        for i, n in enumerate(STEP_OPS):
            per_op_ms[n] += marks[i].elapsed_time(marks[i + 1])
    per_op_ms = {n: v / K for n, v in per_op_ms.items()}
    if split:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())

    extras = world == 1   # the single-GPU diagnostics below are not repeated per rank
    # ---- C1: latency-bound; us per call over back-to-back launches
    c1src = torch.from_numpy(host["C1"]["src"]).to(dev)
    c1dst = torch.empty(host["C1"]["dst_shape"], dtype=torch.float64, device=dev)
    for _ in range(10):
        T.embed(c1dst, c1src)
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ea.record(stream)
    n_c1 = 200
    for _ in range(n_c1):
        T.embed(c1dst, c1src)
    eb.record(stream)
    torch.cuda.synchronize(dev)
    c1_us = ea.elapsed_time(eb) * 1000.0 / n_c1
    # the same call with its arguments marshalled once (triot.prepare_embed)
    c1_call = T.prepare_embed(c1dst, c1src)
    for _ in range(10):
        c1_call()
    ea.record(stream)
    for _ in range(n_c1):
        c1_call()
    eb.record(stream)
    torch.cuda.synchronize(dev)
    c1_prepared_us = ea.elapsed_time(eb) * 1000.0 / n_c1
    # the same 200 calls captured once in a CUDA graph: device-side us per op (no host cost)
    c1_graph_us = None
    try:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for _ in range(n_c1):
                T.embed(c1dst, c1src)
        graph.replay()
        torch.cuda.synchronize(dev)
        ea.record(stream)
        for _ in range(5):
            graph.replay()
        eb.record(stream)
        torch.cuda.synchronize(dev)
        c1_graph_us = ea.elapsed_time(eb) * 1000.0 / (5 * n_c1)
    except Exception as exc:  # graph capture unavailable: report the host-bound number only
        c1_graph_us = f"unavailable: {exc}"
    # launch floor of the same run: a one-element torch fill (one tiny kernel per call)
    z1 = torch.empty(1, dtype=torch.float64, device=dev)
    for _ in range(10):
        z1.fill_(0.0)
    ea.record(stream)
    for _ in range(n_c1):
        z1.fill_(0.0)
    eb.record(stream)
    torch.cuda.synchronize(dev)
    floor_us = ea.elapsed_time(eb) * 1000.0 / n_c1
    floor_graph_us = None
    try:
        gz = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gz):
            for _ in range(n_c1):
                z1.fill_(0.0)
        gz.replay()
        torch.cuda.synchronize(dev)
        ea.record(stream)
        for _ in range(5):
            gz.replay()
        eb.record(stream)
        torch.cuda.synchronize(dev)
        floor_graph_us = round(ea.elapsed_time(eb) * 1000.0 / (5 * n_c1), 3)
        del gz
    except Exception as exc:
        floor_graph_us = f"unavailable: {exc}"

    # ---- each op alone after a clean L2 scrub (write a 512 MB buffer, then read another so
    # every dirty line is written back before the timed launch): median of 5 single launches
    iso, graph20, ev_context = {}, {}, {}
    if extras and not args.no_isolated:
        scratch = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
        clean = torch.ones(512 << 18, dtype=torch.int32, device=dev)
        fns = {"C2": lambda: T.embed(g["dst2"], g["src2"]),
               "C3": lambda: T.expected_value(g["p3"], out=g["m3"]),
               "C4": lambda: T.apply_binary(g["a4"], g["b4"], "mul", out=g["c4"]),
               "C5": lambda: T.embed(g["dst5"], g["src5"])}
        for n, fn in fns.items():
            ts = []
            for _ in range(args.iso_reps):   # event timestamps are quantised (~2 us here)
                scratch.fill_(1)
                clean.sum()
                ea.record(stream)
                fn()
                eb.record(stream)
                torch.cuda.synchronize(dev)
                ts.append(ea.elapsed_time(eb))
            iso[n] = ts
        # cross-check (steady state): 20 back-to-back launches captured in one CUDA graph, no
        # scrub -- working sets >> L2, so each launch pays its predecessor's write-back
        for n, fn in fns.items():
            try:
                gr = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gr):
                    for _ in range(20):
                        fn()
                gr.replay()
                torch.cuda.synchronize(dev)
                ea.record(stream)
                gr.replay()
                eb.record(stream)
                torch.cuda.synchronize(dev)
                graph20[n] = ea.elapsed_time(eb) / 20
                del gr
            except Exception as exc:
                graph20[n] = f"unavailable: {exc}"
        # context for C3 (134 MB, one launch: launch, ramp and tail are not amortised): the same
        # kernel instance (d = 6, f64, power-of-two extents) on a PMF 8x the size, and a library
        # reduction (torch.sum, one value out) over C3's own bytes, both under both protocols
        try:
            p8 = torch.rand((32, 32, 32, 16, 16, 16), dtype=torch.float64, device=dev)
            m8 = torch.empty(6, dtype=torch.float64, device=dev)
            s3 = torch.empty((), dtype=torch.float64, device=dev)
            p3flat = g["p3"].view(-1)
            ctx = {"EV d=6 f64 (32,32,32,16,16,16), 1.07 GB":
                   (lambda: T.expected_value(p8, out=m8), p8.numel() * 8 + 48),
                   "torch.sum over C3's p (134 MB, library reduction)":
                   (lambda: torch.sum(p3flat, dim=(0,), out=s3), g["p3"].numel() * 8 + 8)}
            for n, (fn, nbytes) in ctx.items():
                fn()
                ts = []
                for _ in range(15):
                    scratch.fill_(1)
                    clean.sum()
                    ea.record(stream)
                    fn()
                    eb.record(stream)
                    torch.cuda.synchronize(dev)
                    ts.append(ea.elapsed_time(eb))
                gr = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gr):
                    for _ in range(20):
                        fn()
                gr.replay()
                torch.cuda.synchronize(dev)
                ea.record(stream)
                gr.replay()
                eb.record(stream)
                torch.cuda.synchronize(dev)
                g20 = ea.elapsed_time(eb) / 20
                ms = statistics.median(ts)
                ev_context[n] = {"bytes": nbytes, "us": round(ms * 1000, 2),
                                 "gbs": round(nbytes / (ms * 1e-3) / 1e9, 1),
                                 "graph20_us": round(g20 * 1000, 2),
                                 "graph20_gbs": round(nbytes / (g20 * 1e-3) / 1e9, 1)}
                del gr
            del p8, m8
        except Exception as exc:
            ev_context["unavailable"] = str(exc)
        del scratch, clean

    # ---- the paper's own Benchmarks 1-3 (§8(f) NEXT-2/3), same isolated protocol
    paper = {}
    if extras and not args.no_isolated:
        from triot_inputs import make_paper_inputs
        scratch = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
        clean = torch.ones(512 << 18, dtype=torch.int32, device=dev)
        b1 = make_paper_inputs("B1")
        y1 = torch.from_numpy(b1["src"]).to(dev)
        x1 = torch.empty(b1["dst_shape"], dtype=torch.float64, device=dev)
        b2 = make_paper_inputs("B2")
        a2, bb2 = torch.from_numpy(b2["a"]).to(dev), torch.from_numpy(b2["b"]).to(dev)
        o2 = torch.empty(1, dtype=torch.float64, device=dev)
        b3 = make_paper_inputs("B3")
        x3 = torch.from_numpy(b3["x"]).to(dev)
        y3, z3 = torch.from_numpy(b3["y"]).to(dev), torch.from_numpy(b3["z"]).to(dev)
        n1 = math.prod(b1["dst_shape"]) * 8
        n3 = math.prod(b3["x"].shape) * 8
        cases = {"B1 crop copy": (lambda: T.embed(x1, y1), 2 * n1),
                 "B2 inner product": (lambda: T.inner_product(a2, bb2, out=o2), 2 * n1 + 8),
                 "B3 fused update": (lambda: T.fused_update(x3, y3, z3), 4 * n3)}
        for name, (fn, nbytes) in cases.items():
            fn()
            ts = []
            for _ in range(15):
                scratch.fill_(1)
                clean.sum()
                ea.record(stream)
                fn()
                eb.record(stream)
                torch.cuda.synchronize(dev)
                ts.append(ea.elapsed_time(eb))
            ms = statistics.fmean(ts)
            gbs = nbytes / (ms * 1e-3) / 1e9
            paper[name] = {"bytes": nbytes, "us": round(ms * 1000, 2), "gbs": round(gbs, 1),
                           "pct_of_8000": round(100 * gbs / NOMINAL_HBM_GBS, 1)}
        # Benchmark 4: naive 2-D convolution of two (2^8, 2^3) matrices --
        # latency-bound (7,665 sequential sums of up to 2,048 rounded products), so reported
        # as time and multiply-adds per second next to the oracle's time, not as HBM bandwidth
        rng4 = np.random.default_rng(17)
        l4 = torch.from_numpy(rng4.random((256, 8))).to(dev)
        r4 = torch.from_numpy(rng4.random((256, 8))).to(dev)
        o4 = torch.empty((511, 15), dtype=torch.float64, device=dev)
        T.naive_convolve(l4, r4, out=o4)
        ea.record(stream)
        for _ in range(20):
            T.naive_convolve(l4, r4, out=o4)
        eb.record(stream)
        torch.cuda.synchronize(dev)
        us4 = ea.elapsed_time(eb) * 1000 / 20
        macs = 256 * 8 * 256 * 8
        paper["B4 naive convolution"] = {
            "macs": macs, "us": round(us4, 2), "gmacs_per_s": round(macs / us4 / 1e3, 1),
            "bound": "latency (sequential per-output sums, bit-exact order)"}
        del scratch, clean, y1, x1, a2, bb2, x3, y3, z3

    # ---- e2e: same step through the public API with pinned HOST buffers; every step copies
    # its inputs H2D and reads its results back D2H inside the timed region
    e2e = run_e2e(args, sl, dev, stream, T, world, rank, split)
    sampler.stop()

    peak, peak_kind = measured_peak()
    step_bytes = sum(algorithmic_bytes(n) for n in STEP_OPS)
    # strong scaling: the ranks together process ONE global instance per step
    value = K * step_bytes / (total_ms * 1e-3) / 1e9
    per_op = []
    for n in STEP_OPS:
        b = algorithmic_bytes(n)
        gbs = b / (per_op_ms[n] * 1e-3) / 1e9
        per_op.append({"config": n, "op": {"C2": "embed", "C3": "expected_value",
                                          "C4": "apply_binary", "C5": "embed"}[n],
                       "bytes": b, "us": round(per_op_ms[n] * 1000, 2), "gbs": round(gbs, 1),
                       "pct_of_8000": round(100 * gbs / NOMINAL_HBM_GBS, 1),
                       "pct_of_measured": round(100 * gbs / peak, 1)})
    per_op_iso = []
    for n, ts in iso.items():
        b = algorithmic_bytes(n)
        ms = statistics.median(ts)
        gbs = b / (ms * 1e-3) / 1e9
        row = {"config": n, "us": round(ms * 1000, 2), "gbs": round(gbs, 1),
               "pct_of_8000": round(100 * gbs / NOMINAL_HBM_GBS, 1),
               "pct_of_measured": round(100 * gbs / peak, 1),
               "us_min_median_mean_max": [round(min(ts) * 1000, 2), round(ms * 1000, 2),
                                          round(statistics.fmean(ts) * 1000, 2),
                                          round(max(ts) * 1000, 2)]}
        g20 = graph20.get(n)
        if isinstance(g20, float):
            row["graph20_us"] = round(g20 * 1000, 2)
            row["graph20_gbs"] = round(b / (g20 * 1e-3) / 1e9, 1)
        per_op_iso.append(row)
    dom = max(per_op, key=lambda r: r["us"])
    traffic, traffic_src = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f)
        traffic = tj.get(dom["config"])
        traffic_src = ("profiles/traffic.json: " + str(tj.get("_source", "")) +
                       " (not this run: ncu replays kernels and is never run inside the bench)")
    except Exception:
        traffic = None
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(budget_s=args.cpu_budget)
        if "B4 naive convolution" in paper:  # the oracle's time for Benchmark 4, same leg
            paper["B4 naive convolution"]["oracle_us_1core"] = cpu.get("b4_oracle_us")
    out = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
        "steps": K, "warmup": args.warmup, "ms_per_step": round(total_ms / K, 4),
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None,
        "dtype": "f32+f64 (embed: raw 32-bit words; binary f64; EV f64 accumulate)",
        "data": "synthetic (numpy PCG64 seeds 1..5, BASELINE.json configs)",
        "config": {"workload": WORKLOAD, "bytes_per_step": step_bytes,
                   "ops": "C2 embed f32 (384)^3->(512)^3; C3 EV f64 (16)^6; C4 mul f64 "
                          "(32,48,24,40,36)x(40,32,32,32,32)->(32,32,24,32,32); C5 embed f32 "
                          "(3)^14->(4)^14",
                   "l2": "no flush: 2.6 GB per step >> 126 MB L2, each op's inputs evicted "
                         "by its predecessor",
                   "parallelism": ("single GPU" if world == 1 else
                                   f"outer-loop partition over {world} GPUs (P:607): embed / "
                                   "binary boxes with no collective, EV all_gather of 6 doubles "
                                   "+ rank-order triot_sum_rows")},
        "per_op": per_op,
        "per_op_isolated": {"note": f"each op alone after a clean L2 scrub, {args.iso_reps} "
                                    "launches: us = median (event timestamps are quantised to "
                                    "~2 us); graph20 = 20 back-to-back launches in one CUDA "
                                    "graph, no scrub (steady state incl. write-back)",
                            "ops": per_op_iso,
                            "c3_context": ev_context},
        "paper_benchmarks": {"note": "P:333 Benchmarks 1-3 at the paper's shapes, f64, "
                                     "isolated as per_op_isolated (B3 is 27 MB: launch-bound)",
                             "ops": paper},
        "c1_latency_us": {"per_call_host_bound": round(c1_us, 2),
                          "per_call_prepared": round(c1_prepared_us, 2),
                          "per_op_in_cuda_graph": (round(c1_graph_us, 3)
                                                   if isinstance(c1_graph_us, float)
                                                   else c1_graph_us),
                          "bytes": algorithmic_bytes("C1"),
                          "launch_floor_1elem_fill": {"per_call": round(floor_us, 2),
                                                      "per_op_in_cuda_graph": floor_graph_us}},
        "roofline": {"bound": "hbm", "kernel": f"{dom['op']} ({dom['config']})",
                     "achieved": dom["gbs"], "peak": peak, "unit": "GB/s",
                     "frac": round(dom["gbs"] / peak, 3), "peak_kind": peak_kind,
                     "traffic": traffic, "traffic_source": traffic_src},
        "clocks": sampler.summary(),
        "e2e": e2e,
        "gpu_launches": (5 if split else 4) * K,
        "cpu_baseline": cpu,
    }
    if split:
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(out), flush=True)


def slab_plan(host, world, rank):
    """This rank's part of one global instance of each step config: its box of the counter
    (paper_1608_00099_b200.parallel.leading_box) and the matching input blocks.  At
    world == 1 the box is the whole config."""
    from paper_1608_00099_b200.parallel import leading_box

    def take(arr, box):
        idx = tuple(slice(min(lo, n), min(hi, n)) for (lo, hi), n in zip(box, arr.shape))
        return np.ascontiguousarray(arr[idx])

    plan = {}
    for n in ("C2", "C5"):
        dsh = host[n]["dst_shape"]
        box = leading_box(dsh, world, rank)
        plan[n] = {"box": box, "dst_shape": tuple(hi - lo for lo, hi in box),
                   "src": take(host[n]["src"], box)}
    p = host["C3"]["p"]
    box = leading_box(p.shape, world, rank)
    plan["C3"] = {"box": box, "p": take(p, box), "offset": tuple(lo for lo, _ in box)}
    ish = host["C4"]["iter_shape"]
    box = leading_box(ish, world, rank)
    ab = [(lo, hi) for lo, hi in box]
    a4, b4 = host["C4"]["a"], host["C4"]["b"]
    # a and b keep their own extents outside the box's cut axes (each indexed by its own shape)
    cut = [k for k, (lo, hi) in enumerate(ab) if (lo, hi) != (0, ish[k])]
    boxa = [ab[k] if k in cut else (0, a4.shape[k]) for k in range(a4.ndim)]
    boxb = [ab[k] if k in cut else (0, b4.shape[k]) for k in range(b4.ndim)]
    plan["C4"] = {"box": box, "iter_shape": tuple(hi - lo for lo, hi in box),
                  "a": take(a4, boxa), "b": take(b4, boxb)}
    return plan


def pcie_floors(dev, h2d_bytes, d2h_bytes):
    """PCIe copy rates of this box in the same run (pinned host <-> device, torch copies): H2D
    alone, D2H alone and both at once on two streams; floor_ms = the step's copies at those
    rates (the e2e value cannot beat it)."""
    import torch
    n = 256 << 20
    hs = torch.empty(n, dtype=torch.uint8).pin_memory()
    hd = torch.empty(n, dtype=torch.uint8).pin_memory()
    ds = torch.empty(n, dtype=torch.uint8, device=dev)
    dd = torch.empty(n, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def timed(fn, reps=4):
        fn()
        torch.cuda.synchronize(dev)
        t = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize(dev)
        return (time.perf_counter() - t) / reps

    t_h2d = timed(lambda: ds.copy_(hs, non_blocking=True))
    t_d2h = timed(lambda: hd.copy_(dd, non_blocking=True))

    def both():
        with torch.cuda.stream(s1):
            ds.copy_(hs, non_blocking=True)
        with torch.cuda.stream(s2):
            hd.copy_(dd, non_blocking=True)
    t_both = timed(both)
    h2d_gbs, d2h_gbs, both_gbs = n / t_h2d / 1e9, n / t_d2h / 1e9, 2 * n / t_both / 1e9
    floor_ms = 1e3 * max(h2d_bytes / (h2d_gbs * 1e9), d2h_bytes / (d2h_gbs * 1e9),
                         (h2d_bytes + d2h_bytes) / (both_gbs * 1e9))
    del hs, hd, ds, dd
    return {"h2d_gbs": round(h2d_gbs, 1), "d2h_gbs": round(d2h_gbs, 1),
            "both_gbs": round(both_gbs, 1), "floor_ms_per_step": round(floor_ms, 2),
            "how": "256 MiB pinned<->device torch copies, wall clock over 4 reps after 1"}


def run_e2e(args, sl, dev, stream, T, world, rank, split):
    import torch
    import torch.distributed as dist
    pin = {
        "src2": torch.from_numpy(sl["C2"]["src"]).pin_memory(),
        "p3": torch.from_numpy(sl["C3"]["p"]).pin_memory(),
        "a4": torch.from_numpy(sl["C4"]["a"]).pin_memory(),
        "b4": torch.from_numpy(sl["C4"]["b"]).pin_memory(),
        "src5": torch.from_numpy(sl["C5"]["src"]).pin_memory(),
    }
    outs = {
        "dst2": torch.empty(sl["C2"]["dst_shape"], dtype=torch.float32).pin_memory(),
        "m3": torch.empty(6, dtype=torch.float64).pin_memory(),
        "c4": torch.empty(sl["C4"]["iter_shape"], dtype=torch.float64).pin_memory(),
        "dst5": torch.empty(sl["C5"]["dst_shape"], dtype=torch.float32).pin_memory(),
    }
    ish = sl["C4"]["iter_shape"]
    # bytes that cross PCIe per step on this rank: the input blocks (b's rows beyond the
    # iteration shape are not sent by the slab pipeline) and the results
    b4 = sl["C4"]["b"]
    h2d = sum(t.numel() * t.element_size() for t in pin.values()) - \
        (b4.shape[0] - ish[0]) * (b4[0].size * 8 if b4.shape[0] else 0)
    d2h = sum(t.numel() * t.element_size() for t in outs.values())
    staging3 = torch.empty(64 << 20, dtype=torch.uint8, device=dev)
    if split:
        m3d = torch.empty(6, dtype=torch.float64, device=dev)
        g3 = torch.empty(world * 6, dtype=torch.float64, device=dev)
        r3 = torch.empty(6, dtype=torch.float64, device=dev)
        res3 = torch.empty(6, dtype=torch.float64).pin_memory()

    # every leg through the C-ABI host-buffer entry points (triot_embed_host, triot_expected_
    # value_host, triot_apply_binary_host): slabs streamed through device staging with H2D,
    # kernel and D2H overlapped, each op on its own stream so one op's device-to-host
    # drain overlaps the next op's host-to-device feed; the step ends when every stream is done
    side = [torch.cuda.Stream(dev) for _ in range(4)]

    def e2e_step():
        for sd in side:
            sd.wait_stream(stream)
        # issue order: the D2H-heavy leg with a tiny input (C5: 19 MB in, 1.07 GB out) first, so
        # the device-to-host engine starts draining while the others' inputs stream in (B200:
        # 36.9-38.2 ms vs 40-43 ms issuing C2 first, profiles/r02_e2e_slots*.jsonl)
        with torch.cuda.stream(side[3]):
            T.embed_host(outs["dst5"], pin["src5"], device=dev)
        with torch.cuda.stream(side[0]):
            T.embed_host(outs["dst2"], pin["src2"], device=dev)
        with torch.cuda.stream(side[2]):
            T.apply_binary_host(pin["a4"], pin["b4"], "mul", out=outs["c4"], iter_shape=ish,
                                device=dev)
        with torch.cuda.stream(side[1]):
            T.expected_value_host(pin["p3"], staging3, out=outs["m3"],
                                  offset=sl["C3"]["offset"] if split else None)
            if split:   # amalgamate the ranks' results: 48 bytes each way
                m3d.copy_(outs["m3"], non_blocking=True)
                dist.all_gather_into_tensor(g3, m3d)
                T.sum_rows(g3.view(world, 6), out=r3)
                res3.copy_(r3, non_blocking=True)
        for sd in side:
            stream.wait_stream(sd)

    for _ in range(2):   # warm-up: staging rings, pinned pages, copy-engine clocks
        e2e_step()
    torch.cuda.synchronize(dev)
    k = max(1, min(args.steps, args.e2e_steps))
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if split:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ea.record(stream)
    for _ in range(k):
        e2e_step()
    eb.record(stream)
    torch.cuda.synchronize(dev)
    ms = ea.elapsed_time(eb) / k
    if split:
        import torch as _t
        v = _t.tensor([ms, float(h2d), float(d2h)], dtype=_t.float64, device=dev)
        mx = v[:1].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(v, op=dist.ReduceOp.SUM)
        ms, h2d, d2h = float(mx.item()), int(v[1].item()), int(v[2].item())
    step_bytes = sum(algorithmic_bytes(n) for n in STEP_OPS)
    out = {"value": round(step_bytes / (ms * 1e-3) / 1e9, 2), "unit": UNIT,
           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": k,
           "ms_per_step": round(ms, 3),
           "note": "public C-ABI host-buffer entry points from pinned host memory: "
                   "triot_embed_host, triot_expected_value_host, triot_apply_binary_host "
                   "(chunk-streamed, H2D / kernel / D2H overlapped), one stream per op; every "
                   "input's H2D and every result's D2H inside the timed region"}
    if world == 1:
        out["pcie_same_run"] = pcie_floors(dev, h2d, d2h)
    return out


# ----------------------------------------------------------------------------- oracle arms

def _slab(name: str, frac: float):
    """A leading slab (fraction of axis 0) of config `name`: the bounded CPU sample."""
    inp = make_inputs(name)
    if name in ("C1", "C2", "C5"):
        dsh = inp["dst_shape"]
        m = max(1, int(math.ceil(frac * dsh[0])))
        src = np.ascontiguousarray(inp["src"][:m])
        dst_shape = (m,) + tuple(dsh[1:])
        rd = math.prod(min(a, b) for a, b in zip(src.shape, dst_shape)) * src.itemsize
        wr = math.prod(dst_shape) * src.itemsize
        return ("embed", (src, dst_shape), rd + wr)
    if name == "C3":
        p = inp["p"]
        m = max(1, int(math.ceil(frac * p.shape[0])))
        ps = np.ascontiguousarray(p[:m])
        return ("ev", (ps,), ps.nbytes + ps.ndim * 8)
    ish = inp["iter_shape"]
    m = max(1, int(math.ceil(frac * ish[0])))
    a = np.ascontiguousarray(inp["a"][:m])
    b = np.ascontiguousarray(inp["b"][:m])
    ish = (m,) + tuple(ish[1:])
    return ("binary", (a, b, ish), 3 * math.prod(ish) * 8)


def _run_slab(kind, args_):
    from oracle import oracle as O
    if kind == "embed":
        src, dsh = args_
        dst = np.empty(dsh, dtype=src.dtype)
        t = time.perf_counter()
        O.embed(dst, src)
        return time.perf_counter() - t
    if kind == "ev":
        t = time.perf_counter()
        O.expected_value(args_[0])
        return time.perf_counter() - t
    a, b, ish = args_
    t = time.perf_counter()
    O.apply_binary(a, b, "mul", iter_shape=ish)
    return time.perf_counter() - t


def _calibrate(seconds: float) -> float:
    """Fraction of axis 0 whose oracle run takes about `seconds` (per-byte rate of a probe)."""
    probe = [_slab(n, 1.0 / 64) for n in STEP_OPS]
    t = sum(_run_slab(k, a) for k, a, _ in probe)
    pbytes = sum(b for _, _, b in probe)
    full = sum(algorithmic_bytes(n) for n in STEP_OPS)
    full_s = t / max(pbytes, 1) * full
    return min(1.0, seconds / max(full_s, 1e-9))


def cpu_baseline(budget_s: float = 20.0, frac: float | None = None, reps: int = 3):
    """The oracle as it stands, 1 thread, on a slab of each op sized to ~budget_s seconds in
    all: `reps` repetitions (init excluded), min / mean / max reported, value = median."""
    if frac is None:
        frac = _calibrate(budget_s / reps)
    slabs = [_slab(n, frac) for n in STEP_OPS]
    nbytes = sum(b for _, _, b in slabs)
    runs = [sum(_run_slab(k, a) for k, a, _ in slabs) for _ in range(reps)]
    secs = statistics.median(runs)
    # Benchmark 4 (naive convolution) on the same host thread, for the paper-benchmark line
    from oracle import oracle as O
    rng4 = np.random.default_rng(17)
    l4, r4 = rng4.random((256, 8)), rng4.random((256, 8))
    t0 = time.perf_counter()
    O.naive_convolve(l4, r4)
    b4_us = (time.perf_counter() - t0) * 1e6
    return {"value": round(nbytes / secs / 1e9, 4), "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"leading {frac:.3f} of axis 0 of each of C2,C3,C4,C5 (one slab per op), "
                      f"{nbytes} algorithmic bytes, median of {reps} reps, single thread",
            "reps": reps,
            "seconds_min_mean_max": [round(min(runs), 3), round(statistics.fmean(runs), 3),
                                     round(max(runs), 3)],
            "gbs_min_mean_max": [round(nbytes / max(runs) / 1e9, 4),
                                 round(nbytes / statistics.fmean(runs) / 1e9, 4),
                                 round(nbytes / min(runs) / 1e9, 4)],
            "b4_oracle_us": round(b4_us, 1), "host": host_info()}


def host_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        aff = len(os.sched_getaffinity(0))
    except AttributeError:
        aff = None
    return {"cpu_model": model, "cpu_count": os.cpu_count(), "affinity_cores": aff,
            "threads_used": 1}


def run_reference(args, rank, world):
    if rank != 0:
        return
    from oracle import oracle as O
    O.build()
    frac = _calibrate(args.ref_budget / max(1, args.steps + args.warmup))
    slabs = [_slab(n, frac) for n in STEP_OPS]
    step_bytes = sum(b for _, _, b in slabs)
    for _ in range(args.warmup):
        for k, a, _ in slabs:
            _run_slab(k, a)
    total = 0.0
    for _ in range(args.steps):
        total += sum(_run_slab(k, a) for k, a, _ in slabs)
    value = args.steps * step_bytes / total / 1e9
    sample = (f"leading {frac:.4f} of axis 0 of each of C2,C3,C4,C5 per step "
              f"({step_bytes} algorithmic bytes), single thread")
    out = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1000 * total / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "bytes_per_step": step_bytes,
                   "slab": f"leading {frac:.4f} of axis 0 of each of C2, C3, C4, C5 per step "
                           "(a bounded sample of the same configs: the full step would take "
                           "~6 s of oracle time per step)",
                   "parallelism": "CPU oracle, rank 0 only"},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": sample, "host": host_info()},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--e2e-steps", type=int, default=6)
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--ref-budget", type=float, default=120.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-isolated", action="store_true")
    ap.add_argument("--iso-reps", type=int, default=50)
    ap.add_argument("--split-test", action="store_true",
                    help="run the multi-GPU partition path at world size 1 (testing)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and "WORLD_SIZE" in os.environ:
        args.gpus = world
    if world > 1 and "RANK" not in os.environ:
        sys.exit("for --gpus > 1 launch with torch.distributed.run (one process per GPU)")
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
