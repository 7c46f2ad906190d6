"""Summarise an ncu --set full report: per kernel launch, the DRAM/L2/issue metrics we cite.

    python tools/ncu_summary.py report.ncu-rep [--json out.json]
"""
import csv
import io
import json
import subprocess
import sys

WANT = [
    "Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
    "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_write.sum",
    # not in --set full: request them with --metrics (see profiles/README.md)
    "smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.ratio",
    "smsp__sass_average_data_bytes_per_sector_mem_global_op_st.ratio",
    "lts__d_sectors_fill_device.sum", "smsp__cycles_active.avg",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_drain_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "sm__cycles_elapsed.avg.per_second",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
    "smsp__sass_data_bytes_mem_global_op_ld.sum",
]

# algorithmic (read, write) bytes per launch of the BASELINE configs
ALGO = {"C2": (226_492_416, 536_870_912), "C3": (134_217_728, 48),
        "C4": (402_653_184, 201_326_592), "C5": (19_131_876, 1_073_741_824)}


def _bytes(d, key):
    v, u = d.get(key), d.get(key + " [unit]", "byte")
    if not isinstance(v, float):
        return None
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    return v * scale


def evidence(res, configs):
    """SURVEY §8(d)'s ncu evidence per kernel, launches matched to configs in order."""
    out = []
    for d, cfg in zip(res, configs):
        rd, wr = ALGO[cfg]
        dr, dw = _bytes(d, "dram__bytes_read.sum"), _bytes(d, "dram__bytes_write.sum")
        t = d.get("gpu__time_duration.sum")
        tu = d.get("gpu__time_duration.sum [unit]", "us")
        t_s = t * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3}.get(tu, 1e-6)
        req_ld = d.get("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum")
        sec_ld = d.get("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum")
        req_st = d.get("l1tex__t_requests_pipe_lsu_mem_global_op_st.sum")
        sec_st = d.get("l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum")
        nvec = (rd + wr) / 32.0
        out.append({
            "config": cfg, "kernel": d.get("Kernel Name"), "us_cold": round(t_s * 1e6, 2),
            "dram_GBps": round((dr + dw) / t_s / 1e9, 1),
            "dram_pct_of_peak": d.get("dram__throughput.avg.pct_of_peak_sustained_elapsed") or
            d.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "overfetch_read": round(dr / rd, 3) if rd > 1000 else None,
            "write_completeness": round(dw / wr, 3) if wr > 1000 else None,
            "bytes_per_sector_ld": d.get("smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.ratio"),
            "bytes_per_sector_st": d.get("smsp__sass_average_data_bytes_per_sector_mem_global_op_st.ratio"),
            "sectors_per_request_ld": round(sec_ld / req_ld, 2) if req_ld else None,
            "sectors_per_request_st": round(sec_st / req_st, 2) if req_st else None,
            "warp_inst_per_32B_vector": round(d["smsp__inst_executed.sum"] / nvec, 3),
            "issue_active_pct": d.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "stall_long_scoreboard": d.get(
                "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"),
            "registers": d.get("launch__registers_per_thread"),
            "warps_active_pct": d.get("sm__warps_active.avg.pct_of_peak_sustained_active"),
        })
    return out


def summarise(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        d = {}
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                v = r[i]
                try:
                    v = float(v.replace(",", ""))
                except ValueError:
                    pass
                d[w] = v
                if units[i]:
                    d[w + " [unit]"] = units[i]
        res.append(d)
    return res


if __name__ == "__main__":
    res = summarise(sys.argv[1])
    if "--evidence" in sys.argv:   # --evidence C2,C3,C4,C5 --json out.json
        cfgs = sys.argv[sys.argv.index("--evidence") + 1].split(",")
        ev = evidence(res, cfgs)
        print(json.dumps(ev, indent=1))
        if "--json" in sys.argv:
            with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
                json.dump(ev, f, indent=1)
        sys.exit(0)
    for d in res:
        print("----", d.get("Kernel Name"))
        for k, v in d.items():
            if not k.endswith("[unit]") and k != "Kernel Name":
                print(f"   {k} = {v} {d.get(k + ' [unit]', '')}")
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
            json.dump(res, f, indent=1)
