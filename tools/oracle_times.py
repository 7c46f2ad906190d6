"""Full-size CPU-oracle time per BASELINE config on this host (1 thread, init excluded):
3 reps each, min / mean / max seconds (for BASELINE.md §5).  python tools/oracle_times.py"""
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from triot_inputs import make_inputs  # noqa: E402


def main():
    O.build()
    out = {}
    for n in ("C1", "C2", "C3", "C4", "C5"):
        inp = make_inputs(n)
        if n in ("C1", "C2", "C5"):
            dst = np.empty(inp["dst_shape"], dtype=inp["src"].dtype)
            fn = lambda: O.embed(dst, inp["src"])
        elif n == "C3":
            fn = lambda: O.expected_value(inp["p"])
        else:
            fn = lambda: O.apply_binary(inp["a"], inp["b"], "mul", iter_shape=inp["iter_shape"])
        reps = 200 if n == "C1" else 3
        ts = []
        for _ in range(reps):
            t = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t)
        out[n] = {"s_min_mean_max": [round(min(ts), 6), round(statistics.fmean(ts), 6),
                                     round(max(ts), 6)], "reps": reps}
    import platform
    cpu = None
    with open("/proc/cpuinfo") as f:
        for line in f:
            if line.startswith("model name"):
                cpu = line.split(":", 1)[1].strip()
                break
    out["host"] = {"cpu_model": cpu, "cpu_count": os.cpu_count(),
                   "affinity": len(os.sched_getaffinity(0)), "threads_used": 1,
                   "python": platform.python_version()}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
