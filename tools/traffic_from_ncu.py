"""Write profiles/traffic.json (DRAM bytes per launch, read + write, per op) from the ncu --set
full summary tools/ncu_summary.py produced (gpurun_out/ncu_full_ops.json), in profile_ops.py's
launch order.  bench.py reads it for roofline.traffic and names this file as the source.

    python tools/traffic_from_ncu.py gpurun_out/ncu_full_ops.json C2,C3,C4,C5,... round-label
"""
import json
import sys


def main():
    src, ops, label = sys.argv[1], sys.argv[2].split(","), sys.argv[3]
    rows = json.load(open(src))
    rows = rows if isinstance(rows, list) else rows.get("launches", rows)
    if len(rows) != len(ops):
        sys.exit(f"{len(rows)} launches in {src}, {len(ops)} ops named")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}

    def nbytes(r, key):
        v = r.get(key)
        if v is None:
            return None
        return float(v) * scale[r.get(key + " [unit]", "byte")]

    out = {}
    for op, r in zip(ops, rows):
        rd, wr = nbytes(r, "dram__bytes_read.sum"), nbytes(r, "dram__bytes_write.sum")
        if rd is None or wr is None:
            sys.exit(f"no DRAM bytes for {op}: {list(r)[:8]}")
        out[op] = int(round(rd + wr))
    out["_source"] = (f"{label}: ncu --set full --cache-control all --clock-control none of "
                      "tools/profile_ops.py (one launch per op), dram__bytes_read.sum + "
                      "dram__bytes_write.sum per launch, via tools/evidence.sh")
    out["_note"] = ("write bytes stop at the kernel end: dirty lines still in L2 are not "
                    "counted")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
