"""Build libtriot.so (the C-ABI library) in-tree with nvcc for sm_100a.

    python paper_1608_00099_b200/build.py [--force] [--ptxas-v]   (or __graft_entry__.build())

Objects go to paper_1608_00099_b200/build/, the library to paper_1608_00099_b200/libtriot.so
(both git-ignored; the .so travels to the GPU box with the gpurun snapshot).  The kernel
families are instantiated from csrc/inst.cu once per (op, element size, binary op) and compiled
in parallel.  cudart is linked statically, so the library loads without a CUDA runtime on the
library path; it has no torch dependency.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "libtriot.so")
INCLUDE = os.path.join(ROOT, "include")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# --compress-mode=size: the SASS of the ~1,500 kernel instances is stored compressed in the
# fatbins (decompressed by the driver when a kernel is first loaded): 2.6x smaller objects
NVFLAGS = ["-std=c++17", "-O3", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC,-fvisibility=hidden",
           "-I", CSRC, "-I", INCLUDE, "-diag-suppress", "177", "--compress-mode=size"]

# (object name, source, extra defines)
UNITS = [("plan", "plan.cpp", []), ("capi", "capi.cu", []), ("capi_host", "capi_host.cu", [])]
for _esz in (4, 8):
    UNITS.append((f"inst_0_{_esz}_0", "inst.cu", [f"-DTRIOT_INST_OP=0", f"-DTRIOT_INST_ESZ={_esz}"]))
    UNITS.append((f"inst_2_{_esz}_0", "inst.cu", [f"-DTRIOT_INST_OP=2", f"-DTRIOT_INST_ESZ={_esz}"]))
    UNITS.append((f"inst_2_{_esz}_1", "inst.cu", [f"-DTRIOT_INST_OP=2", f"-DTRIOT_INST_ESZ={_esz}",
                                                  "-DTRIOT_INST_BOP=1"]))
    UNITS.append((f"inst_2_{_esz}_2", "inst.cu", [f"-DTRIOT_INST_OP=2", f"-DTRIOT_INST_ESZ={_esz}",
                                                  "-DTRIOT_INST_BOP=2"]))
    UNITS.append((f"inst_3_{_esz}_0", "inst.cu", ["-DTRIOT_INST_OP=3", f"-DTRIOT_INST_ESZ={_esz}"]))
    UNITS.append((f"inst_4_{_esz}_0", "inst.cu", ["-DTRIOT_INST_OP=4", f"-DTRIOT_INST_ESZ={_esz}"]))
    UNITS.append((f"inst_5_{_esz}_0", "inst.cu", ["-DTRIOT_INST_OP=5", f"-DTRIOT_INST_ESZ={_esz}"]))
    for _op in range(4):
        UNITS.append((f"inst_1_{_esz}_{_op}", "inst.cu",
                      [f"-DTRIOT_INST_OP=1", f"-DTRIOT_INST_ESZ={_esz}", f"-DTRIOT_INST_BOP={_op}"]))

HEADERS = [os.path.join(CSRC, h) for h in ("desc.h", "kernels.cuh", "plan.hpp")] + \
    [os.path.join(INCLUDE, "triot.h")]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(p) > t for p in [src, *HEADERS, __file__])


def _compile(unit, force: bool, ptxas_v: bool) -> tuple[str, str]:
    name, src, defs = unit
    srcp = os.path.join(CSRC, src)
    obj = os.path.join(BUILD, name + ".o")
    if not force and not _stale(obj, srcp):
        return obj, ""
    cmd = [nvcc(), *NVFLAGS, *defs, "-c", srcp, "-o", obj + ".tmp"]
    if ptxas_v and src.endswith(".cu"):
        cmd[1:1] = ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {name}:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    os.replace(obj + ".tmp", obj)
    return obj, r.stderr


def build(force: bool = False, ptxas_v: bool = False, jobs: int | None = None,
          verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    jobs = jobs or max(1, os.cpu_count() or 1)
    objs, logs = [], []
    with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
        futs = [ex.submit(_compile, u, force, ptxas_v) for u in UNITS]
        for f in futs:
            o, log = f.result()
            objs.append(o)
            if log:
                logs.append(log)
    if force or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB)
                                                for o in objs):
        tmp = LIB + ".tmp"
        cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs,
               "-Xcompiler", "-fvisibility=hidden", "-Xlinker", "--exclude-libs,ALL"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, LIB)
    if verbose:
        for log in logs:
            sys.stderr.write(log)
    return LIB


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--ptxas-v", action="store_true")
    ap.add_argument("-j", type=int, default=None)
    a = ap.parse_args()
    print(build(force=a.force, ptxas_v=a.ptxas_v, jobs=a.j, verbose=a.ptxas_v))


if __name__ == "__main__":
    main()
