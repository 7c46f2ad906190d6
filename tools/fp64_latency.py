import ctypes, os, subprocess
H = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(H, "libfp64lat.so")
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC", "-o", so, os.path.join(H, "fp64_latency.cu")], check=True)
L = ctypes.CDLL(so)
for n in (2048, 8192):
    c = (ctypes.c_longlong * 3)()
    L.run_chains(n, c)
    print(f"n={n}: dadd {c[0]/n:.1f} cyc/op, dmul+dadd(smem) {c[1]/n:.1f} cyc/op, fadd {c[2]/n:.1f} cyc/op")
