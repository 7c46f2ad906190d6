// kernels.cuh -- sm_100a kernels of the TRIOT hot path.
//
// One template family per op, instantiated for D = 1..16 digits (the compile-time dimension of
// Alg 5/6), element size ESZ in {4, 8}, vector width V (32 B / 16 B / 1 element) and
// index type IDX in {u32, u64}.
//
// Work decomposition ("specializing the classes ... that correspond to the outermost for
// loops" to split work across processors): the counter is flattened in lexicographic order
// ("the ideal order for caching") into W vectors of V elements; a warp owns a contiguous
// run of steps, and in step s lane i handles vector 32*s + i, so every warp instruction covers
// 32 consecutive vectors (1 KB of every dense tensor at V*ESZ = 32 B).
//
// Per lane: the start tuple is decoded ONCE with fast division (the %-and-/ derivation of P:139,
// with a multiply-high instead of '/', since "division and modulo operation are almost always
// slower than multiplication and addition"); each tensor's offset is then Horner's rule
// over its own shape (Alg 2).  Every following step advances the tuple by +32 vectors
// with the odometer of Alg 3, unrolled over the compile-time digit count (Alg 6) with
// an early exit once no carry remains (amortised O(1)); each carry adds a precomputed
// per-tensor delta, so offsets stay exactly equal to Horner of the new tuple.
//
// Kernel families (the plan picks one per call):
//   embed_kernel / binary_kernel          32-B (16-B, 1-element) vectors; embed zero runs
//   embed_shift_kernel / binary_shift_..  the same with stores shifted to the 32-byte grid
//   *_flat_kernel                         flat vectors across rows (longer odd extents; EV)
//   *_rows_kernel / *_rowsw_kernel        row windows: a lane per row in a shared-memory row
//                                         table, or a warp per row (short odd rows, views)
//   ev_kernel / ev_view_kernel / ev_tma   expected value (+ view, + opt-in bulk-copy pipeline)
//   dot_kernel / update_kernel            Benchmarks 2 and 3
//   conv_kernel / conv_lane_kernel        Benchmark 4, Alg 15 naive convolution
#pragma once
#include <cuda.h>  // CUtensorMap (the struct only; the encoder is fetched at run time)
#include <cuda_runtime.h>
#include <stdint.h>

#include "desc.h"

namespace triot {

constexpr int kBlock = TRIOT_BLOCK;

// Optional per-block timeline (tools/ev_probe.cu defines TRIOT_EV_TRACE; never in the library).
#ifdef TRIOT_EV_TRACE
__device__ unsigned long long* g_ev_trace;
__device__ __forceinline__ void ev_trace(int slot) {
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_ev_trace[blockIdx.x * 8 + slot] = t;
    g_ev_trace[blockIdx.x * 8 + 7] = smid;
  }
}
#define TRIOT_TRACE(s) ev_trace(s)
#else
#define TRIOT_TRACE(s)
#endif


// ------------------------------------------------------------------ raw memory access (bits)

template <int NB>
struct Mem;

template <>
struct Mem<32> {
  static __device__ __forceinline__ void ld(const void* p, uint32_t* w) {
    asm volatile(
        "ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]),
          "=r"(w[7])
        : "l"(p));
  }
  static __device__ __forceinline__ void st(void* p, const uint32_t* w) {
    asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p),
                 "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]),
                 "r"(w[7])
                 : "memory");
  }
};
template <>
struct Mem<16> {
  static __device__ __forceinline__ void ld(const void* p, uint32_t* w) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
                 : "l"(p));
  }
  static __device__ __forceinline__ void st(void* p, const uint32_t* w) {
    asm volatile("st.global.L1::no_allocate.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(w[0]),
                 "r"(w[1]), "r"(w[2]), "r"(w[3])
                 : "memory");
  }
};
template <>
struct Mem<8> {
  static __device__ __forceinline__ void ld(const void* p, uint32_t* w) {
    asm volatile("ld.global.nc.v2.b32 {%0,%1}, [%2];" : "=r"(w[0]), "=r"(w[1]) : "l"(p));
  }
  // w = pred ? *p : 0 (the address is formed unconditionally; only the load is predicated)
  static __device__ __forceinline__ void ld_or0(const void* p, bool pred, uint32_t* w) {
    asm volatile(
        "{\n .reg .pred q;\n setp.ne.u32 q, %3, 0;\n mov.b32 %0, 0;\n mov.b32 %1, 0;\n"
        " @q ld.global.nc.v2.b32 {%0,%1}, [%2];\n}"
        : "=r"(w[0]), "=r"(w[1])
        : "l"(p), "r"((uint32_t)pred));
  }
  static __device__ __forceinline__ void st(void* p, const uint32_t* w) {
    asm volatile("st.global.v2.b32 [%0], {%1,%2};" ::"l"(p), "r"(w[0]), "r"(w[1]) : "memory");
  }
};
template <>
struct Mem<4> {
  static __device__ __forceinline__ void ld(const void* p, uint32_t* w) {
    asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(w[0]) : "l"(p));
  }
  static __device__ __forceinline__ void ld_or0(const void* p, bool pred, uint32_t* w) {
    asm volatile(
        "{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n mov.b32 %0, 0;\n"
        " @q ld.global.nc.b32 %0, [%1];\n}"
        : "=r"(w[0])
        : "l"(p), "r"((uint32_t)pred));
  }
  static __device__ __forceinline__ void st(void* p, const uint32_t* w) {
    asm volatile("st.global.b32 [%0], %1;" ::"l"(p), "r"(w[0]) : "memory");
  }
};

// Coherent (non-.nc) loads for operands that may alias the kernel's own output: PTX defines
// ld.global.nc only for data read-only for the kernel's lifetime, and apply_binary allows c == a
// (in place), the fused update writes x in place.  The binary and update kernels load
// through these; embed (src may never overlap dst) and the reductions keep .nc.
template <int NB>
struct MemC;
template <>
struct MemC<32> {
  static __device__ __forceinline__ void ld(const void* p, uint32_t* w) {
    asm volatile(
        "ld.global.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]),
          "=r"(w[7])
        : "l"(p));
  }
};
template <>
struct MemC<16> {
  static __device__ __forceinline__ void ld(const void* p, uint32_t* w) {
    asm volatile("ld.global.L1::no_allocate.v4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
                 : "l"(p));
  }
};
template <>
struct MemC<8> {
  static __device__ __forceinline__ void ld(const void* p, uint32_t* w) {
    asm volatile("ld.global.v2.b32 {%0,%1}, [%2];" : "=r"(w[0]), "=r"(w[1]) : "l"(p));
  }
  static __device__ __forceinline__ void ld_or0(const void* p, bool pred, uint32_t* w) {
    asm volatile(
        "{\n .reg .pred q;\n setp.ne.u32 q, %3, 0;\n mov.b32 %0, 0;\n mov.b32 %1, 0;\n"
        " @q ld.global.v2.b32 {%0,%1}, [%2];\n}"
        : "=r"(w[0]), "=r"(w[1])
        : "l"(p), "r"((uint32_t)pred));
  }
};
template <>
struct MemC<4> {
  static __device__ __forceinline__ void ld(const void* p, uint32_t* w) {
    asm volatile("ld.global.b32 %0, [%1];" : "=r"(w[0]) : "l"(p));
  }
  static __device__ __forceinline__ void ld_or0(const void* p, bool pred, uint32_t* w) {
    asm volatile(
        "{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n mov.b32 %0, 0;\n"
        " @q ld.global.b32 %0, [%1];\n}"
        : "=r"(w[0])
        : "l"(p), "r"((uint32_t)pred));
  }
};
template <bool NC, int NB>
struct MemSel {
  using T = Mem<NB>;
};
template <int NB>
struct MemSel<false, NB> {
  using T = MemC<NB>;
};

// Programmatic dependent launch (sm_90+): every kernel is launched with programmatic stream
// serialization, so it may be scheduled while its predecessor on the stream drains.  It lets
// its own successor be scheduled as soon as all its blocks have started (pdl_trigger), and it
// touches no global memory before pdl_wait -- which returns once the predecessor grid has
// completed and its writes are visible -- so stream order semantics are unchanged.
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// The loop-free paths of warps that own a single step (0: off, for A/B measurements)
#ifndef TRIOT_ONESTEP
#define TRIOT_ONESTEP 1
#endif
// Keeps a value's computation ahead of a following pdl_wait(): volatile asm statements are not
// reordered among themselves, so the operand must be ready before the wait is issued.
__device__ __forceinline__ void pin_before_wait(uint32_t x) { asm volatile("" ::"r"(x)); }
__device__ __forceinline__ void pin_before_wait(uint64_t x) { asm volatile("" ::"l"(x)); }

template <int ESZ, typename IDX>
__device__ __forceinline__ const char* addr(const void* base, IDX off) {
  return (const char*)base + (uint64_t)off * ESZ;
}

template <typename IDX>
__device__ __forceinline__ IDX shfl_idx(IDX v, int src) {
  return __shfl_sync(0xffffffffu, v, src);
}

// ------------------------------------------------------------------ index arithmetic

// q = n / e for an invariant e: Granlund-Montgomery round-up multiply-high (u32), or hardware
// division for the 64-bit path (once per lane, so its cost is immaterial).
template <typename IDX>
__device__ __forceinline__ IDX divq(IDX n, IDX e, uint32_t m, uint32_t s);
template <>
__device__ __forceinline__ uint32_t divq<uint32_t>(uint32_t n, uint32_t, uint32_t m, uint32_t s) {
  uint32_t h = __umulhi(n, m);
  return (h + ((n - h) >> (s & 0xffu))) >> (s >> 8);
}
template <>
__device__ __forceinline__ uint64_t divq<uint64_t>(uint64_t n, uint64_t e, uint32_t, uint32_t) {
  return n / e;
}

// Mixed-radix digits of v (P:139's %-and-/): a mask and a shift per digit when every extent
// is a power of two (d.pow2, uniform), else the multiply-high division.
template <int D, typename IDX>
__device__ __forceinline__ void decode_digits(const Desc<IDX>& d, IDX v, IDX (&u)[D]) {
  if (d.pow2) {
#pragma unroll
    for (int k = D - 1; k >= 1; --k) {
      u[k] = v & (d.ext[k] - IDX(1));
      v >>= d.lg[k];
    }
  } else {
#pragma unroll
    for (int k = D - 1; k >= 1; --k) {
      IDX q = divq<IDX>(v, d.ext[k], d.fdm[k], d.fds[k]);
      u[k] = v - q * d.ext[k];
      v = q;
    }
  }
  u[0] = v;
}

// Decode vector index v into digits, then Horner offsets per tensor (Alg 2) -- for a
// tensor 0 dense in the digit space (d.lin0 != 0) Horner reduces to v * lin0.
template <int D, int NT, bool BOUNDS, typename IDX, bool ALLB = false>
__device__ __forceinline__ void odo_start(const Desc<IDX>& d, IDX v, IDX (&u)[D],
                                          IDX (&off)[NT], uint32_t& oob) {
  decode_digits<D, IDX>(d, v, u);
#pragma unroll
  for (int x = 0; x < NT; ++x) {
    IDX o = 0;
    if (x == 0 && d.lin0) {
      o = v * d.lin0;
    } else {
#pragma unroll
      for (int k = 0; k < D; ++k) o += u[k] * d.t[x].sig[k];
    }
    off[x] = o;
  }
  oob = 0;
  if (BOUNDS) {
#pragma unroll
    for (int k = 0; k < (ALLB ? D : D - 1); ++k) oob |= (uint32_t)(u[k] >= d.bnd[k]) << k;
  }
}

// Offsets (Alg 2, Horner per tensor) and bounds of a known tuple -- odo_start without the
// division step, for a tuple obtained by a carry.
template <int D, int NT, bool BOUNDS, typename IDX>
__device__ __forceinline__ void odo_horner(const Desc<IDX>& d, const IDX (&u)[D], IDX (&off)[NT],
                                           uint32_t& oob) {
#pragma unroll
  for (int x = 0; x < NT; ++x) {
    IDX o = 0;
#pragma unroll
    for (int k = 0; k < D; ++k) o += u[k] * d.t[x].sig[k];
    off[x] = o;
  }
  oob = 0;
  if (BOUNDS) {
#pragma unroll
    for (int k = 0; k < D - 1; ++k) oob |= (uint32_t)(u[k] >= d.bnd[k]) << k;
  }
}

// +32 vectors: Alg 3's carry loop, unrolled over the D digits (Alg 6) with early exit.
template <int D, int NT, bool BOUNDS, typename IDX, bool ALLB = false>
__device__ __forceinline__ void odo_step(const Desc<IDX>& d, IDX (&u)[D], IDX (&off)[NT],
                                         uint32_t& oob) {
#pragma unroll
  for (int x = 0; x < NT; ++x) off[x] += d.t[x].step;
  bool carry = false;
#pragma unroll
  for (int k = D - 1; k >= 0; --k) {
    if (k > d.khi) continue;  // digits inside the step: no increment, no incoming carry
    IDX nu = u[k] + d.dlt[k] + (carry ? IDX(1) : IDX(0));
    carry = nu >= d.ext[k];
    if (carry) {
      nu -= d.ext[k];
#pragma unroll
      for (int x = 0; x < NT; ++x) off[x] += d.t[x].kap[k];
    }
    u[k] = nu;
    if (BOUNDS && (ALLB || k < D - 1))
      oob = (oob & ~(1u << k)) | ((uint32_t)(nu >= d.bnd[k]) << k);
    if (k <= d.klo && !carry) break;  // "No more carry operations" (Alg 3)
  }
}

// +1 element: Alg 3 itself -- increment the last digit, carry while it overflows --
// with every tensor offset kept equal to Horner of the new tuple (flat vectors).
template <int D, int NT, bool BOUNDS, typename IDX>
__device__ __forceinline__ void odo_inc1(const Desc<IDX>& d, IDX (&u)[D], IDX (&off)[NT],
                                         uint32_t& oob) {
#pragma unroll
  for (int x = 0; x < NT; ++x) off[x] += d.t[x].sig[D - 1];
#pragma unroll
  for (int k = D - 1; k >= 0; --k) {
    IDX nu = u[k] + 1;
    const bool carry = k > 0 && nu >= d.ext[k];
    if (carry) {
      nu = 0;
#pragma unroll
      for (int x = 0; x < NT; ++x) off[x] += d.t[x].kap[k];
    }
    u[k] = nu;
    if (BOUNDS) oob = (oob & ~(1u << k)) | ((uint32_t)(nu >= d.bnd[k]) << k);
    if (!carry) break;
  }
}

// end of warp's window: min(base0 + wspan, W), guarding wrap-around of the index type
template <typename IDX>
__device__ __forceinline__ IDX warp_end(const Desc<IDX>& d, IDX base0) {
  IDX e = base0 + d.wspan;
  return (e > d.nvec || e < base0) ? d.nvec : e;
}

// element e of a vector: row r = e >> lgL, column c = e & (L-1); offset off + r*rho + c*tau
template <typename IDX>
__device__ __forceinline__ IDX elem_off(IDX off, int e, uint32_t lgL, IDX rho, IDX tau) {
  IDX r = (IDX)((uint32_t)e >> lgL);
  IDX c = (IDX)((uint32_t)e & ((1u << lgL) - 1u));
  return off + r * rho + c * tau;
}

template <int ESZ, int V, typename IDX, bool NC = true>
__device__ __forceinline__ void load_vec(const TensorAcc<IDX>& t, IDX off, uint32_t lgL,
                                         uint32_t* w) {
  constexpr int EW = ESZ / 4;
  if (V > 1 && t.vec) {
    MemSel<NC, V * ESZ>::T::ld(addr<ESZ>(t.ptr, off), w);
  } else {
#pragma unroll
    for (int e = 0; e < V; ++e)
      MemSel<NC, ESZ>::T::ld(addr<ESZ>(t.ptr, elem_off(off, e, lgL, t.rho, t.tau)), w + e * EW);
  }
}

template <int ESZ, int V, typename IDX>
__device__ __forceinline__ void store_vec(const TensorAcc<IDX>& t, IDX off, uint32_t lgL,
                                          const uint32_t* w) {
  constexpr int EW = ESZ / 4;
  if (V > 1 && t.vec) {
    Mem<V * ESZ>::st((void*)addr<ESZ>(t.ptr, off), w);
  } else {
#pragma unroll
    for (int e = 0; e < V; ++e)
      Mem<ESZ>::st((void*)addr<ESZ>(t.ptr, elem_off(off, e, lgL, t.rho, t.tau)), w + e * EW);
  }
}

// ------------------------------------------------------------------ embed
// dst[t] = (t < src_shape) ? src[t] : +0.0 over the counter.
// Tensor 0 = dst, tensor 1 = src.  Raw 32-bit words are moved; no floating point.

template <int D, int ESZ, int V, typename IDX, int K, bool ZR>
__global__ void __launch_bounds__(kBlock) embed_kernel(const __grid_constant__ Desc<IDX> d) {
  constexpr int EW = ESZ / 4;
  constexpr int NW = V * EW;
  const int lane = threadIdx.x & 31;
  const IDX warp = (IDX)blockIdx.x * (kBlock / 32) + (IDX)(threadIdx.x >> 5);
  const IDX base0 = warp * d.wmul;
  pdl_trigger();
  if (base0 >= d.nvec) return;
  const IDX vend = warp_end(d, base0);
  IDX u[D], off[2];
  uint32_t oob;
  IDX v = base0 + (IDX)lane;
  odo_start<D, 2, true, IDX>(d, v, u, off, oob);
  const uint32_t lgL = d.lgL;
  if (TRIOT_ONESTEP && !ZR && d.wspan == 32) {
    // One step per warp (small, launch-bound ops: C1): no loop, no odometer step, and the
    // vector's classification is formed before the wait, so that after it only the loads and
    // the store remain (C1: 1.57 -> 1.18 us per op back to back in a CUDA graph,
    // tools/latency_probe.py, profiles/r02_latency_graph2.jsonl).
    const IDX uv = u[D - 1];
    const bool valid = v < vend;
    const bool any = oob == 0 && uv < d.vany;
    const bool fullv = any && uv < d.vfull;
    const IDX row0 = uv * d.rowmul, col0 = uv * d.colmul;
    const IDX o0 = off[0], o1 = off[1];
    pin_before_wait(o0);
    pin_before_wait(o1);
    pin_before_wait(row0);
    pin_before_wait(col0);
    pin_before_wait((uint32_t)valid | ((uint32_t)any << 1) | ((uint32_t)fullv << 2));
    pdl_wait();
    if (!valid) return;
    uint32_t w[NW];
    if (fullv) {
      load_vec<ESZ, V, IDX>(d.t[1], o1, lgL, w);
    } else {
#pragma unroll
      for (int q = 0; q < NW; ++q) w[q] = 0u;
      if (any) {
#pragma unroll
        for (int e = 0; e < V; ++e) {
          const IDX r = (IDX)((uint32_t)e >> lgL);
          const IDX c = (IDX)((uint32_t)e & ((1u << lgL) - 1u));
          if (row0 + r < d.srows && col0 + c < d.scols)
            Mem<ESZ>::ld(addr<ESZ>(d.t[1].ptr, o1 + r * d.t[1].rho + c * d.t[1].tau), w + e * EW);
        }
      }
    }
    store_vec<ESZ, V, IDX>(d.t[0], o0, lgL, w);
    return;
  }
  pdl_wait();
  IDX b = base0;
  for (;;) {
    while (b < vend && !(ZR && (oob & d.zmask))) {
      b += K * d.dv;
      uint32_t buf[K][NW];
      IDX doff[K];
      bool valid[K];
#pragma unroll
      for (int j = 0; j < K; ++j) {
        valid[j] = v < vend;
        v += d.dv;
        doff[j] = off[0];
        if (valid[j]) {
          const IDX uv = u[D - 1];
          const bool any = oob == 0 && uv < d.vany;
          if (any && uv < d.vfull) {
            load_vec<ESZ, V, IDX>(d.t[1], off[1], lgL, buf[j]);
          } else if (!any) {
#pragma unroll
            for (int q = 0; q < NW; ++q) buf[j][q] = 0u;
          } else {
            // partial vector: per-element bounds (rows of a collapsed vector, columns at the
            // src edge)
            const IDX row0 = uv * d.rowmul, col0 = uv * d.colmul;
#pragma unroll
            for (int e = 0; e < V; ++e) {
              const IDX r = (IDX)((uint32_t)e >> lgL);
              const IDX c = (IDX)((uint32_t)e & ((1u << lgL) - 1u));
              if (row0 + r < d.srows && col0 + c < d.scols) {
                Mem<ESZ>::ld(addr<ESZ>(d.t[1].ptr, off[1] + r * d.t[1].rho + c * d.t[1].tau),
                             buf[j] + e * EW);
              } else {
#pragma unroll
                for (int q = 0; q < EW; ++q) buf[j][e * EW + q] = 0u;
              }
            }
          }
        }
        // past the warp's range the odometer is never read again (the loop ends): skip it
        if (valid[j]) odo_step<D, 2, true, IDX>(d, u, off, oob);
      }
#pragma unroll
      for (int j = 0; j < K; ++j)
        if (valid[j]) store_vec<ESZ, V, IDX>(d.t[0], doff[j], lgL, buf[j]);
    }
    if (!ZR || b >= vend) break;
    // zero run (warp-uniform: digits 0..khi are the same in every lane).  m = the most
    // significant out-of-bounds digit; it stays out of bounds until digits m..khi wrap, i.e.
    // for N - S more steps (N, S = size and mixed-radix value of the sub-counter m..khi).
    const int m = __ffs(oob & d.zmask) - 1;
    // N - S with S = the value of digits m..khi = (step index) mod N, the step index being b/32
    const IDX N = d.zn[m], T = b >> 5;
    IDX run = N - (T - divq<IDX>(T, N, d.zdm[m], d.zds[m]) * N);
    const IDX left = (vend - b + 31) / 32;
    if (run > left) run = left;
    const IDX full = (b + run * 32 <= vend) ? run : run - 1;
    const IDX st0 = d.t[0].step;
    IDX o = off[0];
    uint32_t z[NW];
#pragma unroll
    for (int q = 0; q < NW; ++q) z[q] = 0u;
#pragma unroll 1
    for (IDX r = 0; r < full; ++r, o += st0) store_vec<ESZ, V, IDX>(d.t[0], o, lgL, z);
    if (full < run && v + full * 32 < vend) store_vec<ESZ, V, IDX>(d.t[0], o, lgL, z);
    b += run * 32;
    v += run * 32;
    if (b >= vend) break;
    // the run ended because digits m..khi wrapped: they restart at 0 and digit m-1 takes the
    // carry (Alg 3) -- no re-decode; m >= 1 here (digit 0 wrapping is the end)
#pragma unroll
    for (int k = 0; k < D - 1; ++k)
      if (k >= m && k <= d.khi) u[k] = 0;
    bool cy = true;
#pragma unroll
    for (int k = D - 2; k >= 0; --k) {
      if (k < m && cy) {
        const IDX nu = u[k] + 1;
        cy = k > 0 && nu >= d.ext[k];
        u[k] = cy ? IDX(0) : nu;
      }
    }
    odo_horner<D, 2, true, IDX>(d, u, off, oob);
  }
}

// Shifted stores for an output dense in the counter whose base is misaligned by s elements
// (0 < s < V): a warp step's 32 vectors (one per lane, lane-ordered) are 1 KB contiguous of dst
// starting s elements past a 32-byte boundary.  Lane l >= 1 stores the aligned 32-byte chunk l
// made of lane l-1's last s elements (a shuffle) and its own first V - s; lane 0 stores its
// head and lane 31 its tail element by element (the step's two partial chunks).
template <int ESZ>
__device__ __forceinline__ void store_shifted(char* a0, const uint32_t (&w)[8], int sw,
                                              int lane, int nvalid = 32) {
  constexpr int EW = ESZ / 4;
  uint32_t prev[8], out[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) prev[q] = __shfl_up_sync(0xffffffffu, w[q], 1);
  switch (sw) {  // shift in 32-bit words (uniform)
#define TRIOT_SHIFT_CASE(S)                                                      \
  case S:                                                                        \
    _Pragma("unroll") for (int q = 0; q < 8; ++q) out[q] = q < S ? prev[8 - S + q] : w[q - S]; \
    break;
    TRIOT_SHIFT_CASE(1)
    TRIOT_SHIFT_CASE(2)
    TRIOT_SHIFT_CASE(3)
    TRIOT_SHIFT_CASE(4)
    TRIOT_SHIFT_CASE(5)
    TRIOT_SHIFT_CASE(6)
    default:
    TRIOT_SHIFT_CASE(7)
#undef TRIOT_SHIFT_CASE
  }
  char* al = a0 - sw * 4;  // the 32-byte boundary below lane 0's vector
  if (lane >= 1 && lane < nvalid) {
    Mem<32>::st(al + 32 * lane, out);
  } else if (lane == 0) {
#pragma unroll
    for (int q = 0; q < 8; q += EW)
      if (q < 8 - sw) Mem<ESZ>::st(a0 + q * 4, w + q);
  }
  if (lane == nvalid - 1) {  // the last valid lane's tail: the partial chunk past it
#pragma unroll
    for (int q = 0; q < 8; q += EW)
      if (q >= 8 - sw) Mem<ESZ>::st(al + 32 * nvalid + (q - (8 - sw)) * 4, w + q);
  }
}

// embed into a dst dense in the counter but misaligned (plan dshift): embed_kernel's loads,
// store_shifted for every full warp step, element stores for a ragged last step.
template <int D, int ESZ, typename IDX, int K>
__global__ void __launch_bounds__(kBlock) embed_shift_kernel(const __grid_constant__ Desc<IDX> d) {
  constexpr int V = 32 / ESZ;
  constexpr int EW = ESZ / 4;
  constexpr int NW = V * EW;
  const int lane = threadIdx.x & 31;
  const IDX warp = (IDX)blockIdx.x * (kBlock / 32) + (IDX)(threadIdx.x >> 5);
  const IDX base0 = warp * d.wmul;
  pdl_trigger();
  if (base0 >= d.nvec) return;
  const IDX vend = warp_end(d, base0);
  IDX u[D], off[2];
  uint32_t oob;
  IDX v = base0 + (IDX)lane;
  odo_start<D, 2, true, IDX>(d, v, u, off, oob);
  const uint32_t lgL = d.lgL;
  const int sw = (int)d.dshift * EW;
  pdl_wait();
  for (IDX b = base0; b < vend; b += K * d.dv) {
    uint32_t buf[K][NW];
    IDX doff[K];
    bool valid[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      valid[j] = v < vend;
      v += d.dv;
      doff[j] = off[0];
      if (valid[j]) {
        const IDX uv = u[D - 1];
        const bool any = oob == 0 && uv < d.vany;
        if (any && uv < d.vfull) {
          load_vec<ESZ, V, IDX>(d.t[1], off[1], lgL, buf[j]);
        } else if (!any) {
#pragma unroll
          for (int q = 0; q < NW; ++q) buf[j][q] = 0u;
        } else {
          const IDX row0 = uv * d.rowmul, col0 = uv * d.colmul;
#pragma unroll
          for (int e = 0; e < V; ++e) {
            const IDX r = (IDX)((uint32_t)e >> lgL);
            const IDX c = (IDX)((uint32_t)e & ((1u << lgL) - 1u));
            if (row0 + r < d.srows && col0 + c < d.scols) {
              Mem<ESZ>::ld(addr<ESZ>(d.t[1].ptr, off[1] + r * d.t[1].rho + c * d.t[1].tau),
                           buf[j] + e * EW);
            } else {
#pragma unroll
              for (int q = 0; q < EW; ++q) buf[j][e * EW + q] = 0u;
            }
          }
        }
      } else {
#pragma unroll
        for (int q = 0; q < NW; ++q) buf[j][q] = 0u;
      }
      odo_step<D, 2, true, IDX>(d, u, off, oob);
    }
#pragma unroll
    for (int j = 0; j < K; ++j) {
      if (__all_sync(0xffffffffu, valid[j])) {
        // lane 0's vector address: the step's first element (dst offsets are v * V)
        char* a0 = (char*)d.t[0].ptr + (uint64_t)shfl_idx(doff[j], 0) * ESZ;
        store_shifted<ESZ>(a0, buf[j], sw, lane);
      } else if (valid[j]) {
        store_vec<ESZ, V, IDX>(d.t[0], doff[j], lgL, buf[j]);
      }
    }
  }
}

// ------------------------------------------------------------------ binary
// c[t] = a[t] OP b[t] (Alg 9 apply_tensors).  Tensor 0 = c, 1 = a, 2 = b.
// IEEE round-to-nearest, one rounding per element: explicit _rn intrinsics, no contraction.

template <int OP>
__device__ __forceinline__ float bop(float a, float b) {
  if (OP == 0) return __fadd_rn(a, b);
  if (OP == 1) return __fsub_rn(a, b);
  if (OP == 2) return __fmul_rn(a, b);
  return __fdiv_rn(a, b);
}
template <int OP>
__device__ __forceinline__ double bop(double a, double b) {
  if (OP == 0) return __dadd_rn(a, b);
  if (OP == 1) return __dsub_rn(a, b);
  if (OP == 2) return __dmul_rn(a, b);
  return __ddiv_rn(a, b);
}

template <int ESZ>
struct Elem;
template <>
struct Elem<4> {
  using T = float;
  static __device__ __forceinline__ float get(const uint32_t* w) { return __uint_as_float(w[0]); }
  static __device__ __forceinline__ void put(uint32_t* w, float v) { w[0] = __float_as_uint(v); }
};
template <>
struct Elem<8> {
  using T = double;
  static __device__ __forceinline__ double get(const uint32_t* w) {
    return __hiloint2double((int)w[1], (int)w[0]);
  }
  static __device__ __forceinline__ void put(uint32_t* w, double v) {
    w[0] = (uint32_t)__double2loint(v);
    w[1] = (uint32_t)__double2hiint(v);
  }
};

template <int D, int ESZ, int V, typename IDX, int K, int OP>
__global__ void __launch_bounds__(kBlock) binary_kernel(const __grid_constant__ Desc<IDX> d) {
  constexpr int EW = ESZ / 4;
  constexpr int NW = V * EW;
  const int lane = threadIdx.x & 31;
  const IDX warp = (IDX)blockIdx.x * (kBlock / 32) + (IDX)(threadIdx.x >> 5);
  const IDX base0 = warp * d.wmul;
  pdl_trigger();
  if (base0 >= d.nvec) return;
  const IDX vend = warp_end(d, base0);
  IDX u[D], off[3];
  uint32_t oob;
  IDX v = base0 + (IDX)lane;
  odo_start<D, 3, false, IDX>(d, v, u, off, oob);
  const uint32_t lgL = d.lgL;
  if (TRIOT_ONESTEP && d.wspan == 32) {
    // one step per warp (small, launch-bound ops): offsets formed before the wait, then two
    // loads, the op and one store (embed_kernel's one-step path)
    const bool valid = v < vend;
    const IDX o0 = off[0], o1 = off[1], o2 = off[2];
    pin_before_wait(o0);
    pin_before_wait(o1);
    pin_before_wait(o2);
    pin_before_wait((uint32_t)valid);
    pdl_wait();
    if (!valid) return;
    uint32_t wa[NW], wb[NW], r[NW];
    load_vec<ESZ, V, IDX, false>(d.t[1], o1, lgL, wa);
    load_vec<ESZ, V, IDX, false>(d.t[2], o2, lgL, wb);
#pragma unroll
    for (int e = 0; e < V; ++e)
      Elem<ESZ>::put(r + e * EW, bop<OP>(Elem<ESZ>::get(wa + e * EW), Elem<ESZ>::get(wb + e * EW)));
    store_vec<ESZ, V, IDX>(d.t[0], o0, lgL, r);
    return;
  }
  pdl_wait();
  for (IDX b = base0; b < vend; b += K * d.dv) {
    uint32_t ba[K][NW], bb[K][NW];
    IDX coff[K];
    bool valid[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      valid[j] = v < vend;
      v += d.dv;
      coff[j] = off[0];
      if (valid[j]) {
        load_vec<ESZ, V, IDX, false>(d.t[1], off[1], lgL, ba[j]);
        load_vec<ESZ, V, IDX, false>(d.t[2], off[2], lgL, bb[j]);
      }
      odo_step<D, 3, false, IDX>(d, u, off, oob);
    }
#pragma unroll
    for (int j = 0; j < K; ++j) {
      if (!valid[j]) continue;
      uint32_t r[NW];
#pragma unroll
      for (int e = 0; e < V; ++e)
        Elem<ESZ>::put(r + e * EW,
                       bop<OP>(Elem<ESZ>::get(ba[j] + e * EW), Elem<ESZ>::get(bb[j] + e * EW)));
      store_vec<ESZ, V, IDX>(d.t[0], coff[j], lgL, r);
    }
  }
}

// binary into a c dense in the counter but misaligned (plan dshift): binary_kernel with
// store_shifted for every full warp step (in place is safe: a step's loads precede its stores,
// and each element is loaded and stored by the same warp).
template <int D, int ESZ, typename IDX, int K, int OP>
__global__ void __launch_bounds__(kBlock) binary_shift_kernel(const __grid_constant__ Desc<IDX> d) {
  constexpr int V = 32 / ESZ;
  constexpr int EW = ESZ / 4;
  constexpr int NW = V * EW;
  const int lane = threadIdx.x & 31;
  const IDX warp = (IDX)blockIdx.x * (kBlock / 32) + (IDX)(threadIdx.x >> 5);
  const IDX base0 = warp * d.wmul;
  pdl_trigger();
  if (base0 >= d.nvec) return;
  const IDX vend = warp_end(d, base0);
  IDX u[D], off[3];
  uint32_t oob;
  IDX v = base0 + (IDX)lane;
  odo_start<D, 3, false, IDX>(d, v, u, off, oob);
  const uint32_t lgL = d.lgL;
  const int sw = (int)d.dshift * EW;
  pdl_wait();
  for (IDX b = base0; b < vend; b += K * d.dv) {
    uint32_t ba[K][NW], bb[K][NW];
    IDX coff[K];
    bool valid[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      valid[j] = v < vend;
      v += d.dv;
      coff[j] = off[0];
      if (valid[j]) {
        load_vec<ESZ, V, IDX, false>(d.t[1], off[1], lgL, ba[j]);
        load_vec<ESZ, V, IDX, false>(d.t[2], off[2], lgL, bb[j]);
      }
      odo_step<D, 3, false, IDX>(d, u, off, oob);
    }
#pragma unroll
    for (int j = 0; j < K; ++j) {
      uint32_t r[NW];
#pragma unroll
      for (int e = 0; e < V; ++e)
        Elem<ESZ>::put(r + e * EW,
                       bop<OP>(Elem<ESZ>::get(ba[j] + e * EW), Elem<ESZ>::get(bb[j] + e * EW)));
      if (__all_sync(0xffffffffu, valid[j])) {
        char* a0 = (char*)d.t[0].ptr + (uint64_t)shfl_idx(coff[j], 0) * ESZ;
        store_shifted<ESZ>(a0, r, sw, lane);
      } else if (valid[j]) {
        store_vec<ESZ, V, IDX>(d.t[0], coff[j], lgL, r);
      }
    }
  }
}

// ------------------------------------------------------------------ flat vectors (odd extents)
// When no vector width divides the counter's innermost extent (3, 5, 7, 999, ...), a vector is
// V consecutive elements of the flattened counter, crossing rows.  The lane decodes the tuple of
// its vector's first element once, walks the V elements with the +1 odometer (Alg 3), and then
// skips to its next vector with the mixed-radix step.  Tensors dense with the counter (dst of a
// full embed, a dense c, p) are accessed 32 B at a time at flat offset v*V; the others are
// gathered element by element at their own Horner offsets.

template <int D, int ESZ, typename IDX, int K>
__global__ void __launch_bounds__(kBlock) embed_flat_kernel(const __grid_constant__ Desc<IDX> d) {
  constexpr int V = 32 / ESZ;
  constexpr int EW = ESZ / 4;
  constexpr int NW = V * EW;
  const int lane = threadIdx.x & 31;
  const IDX warp = (IDX)blockIdx.x * (kBlock / 32) + (IDX)(threadIdx.x >> 5);
  const IDX base0 = warp * d.wmul;
  pdl_trigger();
  if (base0 >= d.nvec) return;
  const IDX vend = warp_end(d, base0);
  IDX u[D], off[2];
  uint32_t oob;
  IDX v = base0 + (IDX)lane;
  odo_start<D, 2, true, IDX, true>(d, v * (IDX)V, u, off, oob);
  pdl_wait();
  const bool dvec = d.t[0].vec != 0;
  for (IDX b = base0; b < vend; b += K * d.dv) {
    uint32_t buf[K][NW];
    IDX doff[K][V];
    IDX vj[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      vj[j] = v;
      v += d.dv;
#pragma unroll
      for (int e = 0; e < V; ++e) {
        const bool in = vj[j] < vend && vj[j] * (IDX)V + (IDX)e < d.nelem && oob == 0;
        if (in) {
          Mem<ESZ>::ld(addr<ESZ>(d.t[1].ptr, off[1]), buf[j] + e * EW);
        } else {
#pragma unroll
          for (int q = 0; q < EW; ++q) buf[j][e * EW + q] = 0u;
        }
        doff[j][e] = off[0];
        odo_inc1<D, 2, true, IDX>(d, u, off, oob);
      }
      odo_step<D, 2, true, IDX, true>(d, u, off, oob);
    }
#pragma unroll
    for (int j = 0; j < K; ++j) {
      if (vj[j] >= vend) continue;
      const IDX f0 = vj[j] * (IDX)V;
      if (dvec && f0 + (IDX)V <= d.nelem) {
        Mem<32>::st((void*)addr<ESZ>(d.t[0].ptr, f0), buf[j]);
      } else {
#pragma unroll
        for (int e = 0; e < V; ++e)
          if (f0 + (IDX)e < d.nelem)
            Mem<ESZ>::st((void*)addr<ESZ>(d.t[0].ptr, doff[j][e]), buf[j] + e * EW);
      }
    }
  }
}

template <int D, int ESZ, typename IDX, int K, int OP>
__global__ void __launch_bounds__(kBlock) binary_flat_kernel(const __grid_constant__ Desc<IDX> d) {
  constexpr int V = 32 / ESZ;
  constexpr int EW = ESZ / 4;
  constexpr int NW = V * EW;
  const int lane = threadIdx.x & 31;
  const IDX warp = (IDX)blockIdx.x * (kBlock / 32) + (IDX)(threadIdx.x >> 5);
  const IDX base0 = warp * d.wmul;
  pdl_trigger();
  if (base0 >= d.nvec) return;
  const IDX vend = warp_end(d, base0);
  IDX u[D], off[3];
  uint32_t oob;
  IDX v = base0 + (IDX)lane;
  odo_start<D, 3, false, IDX>(d, v * (IDX)V, u, off, oob);
  pdl_wait();
  const bool cvec = d.t[0].vec != 0, avec = d.t[1].vec != 0, bvec = d.t[2].vec != 0;
  for (IDX b = base0; b < vend; b += K * d.dv) {
    uint32_t ba[K][NW], bb[K][NW];
    IDX coff[K][V];
    IDX vj[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      vj[j] = v;
      v += d.dv;
      const IDX f0 = vj[j] * (IDX)V;
      const bool full = vj[j] < vend && f0 + (IDX)V <= d.nelem;
      if (full && avec) MemC<32>::ld(addr<ESZ>(d.t[1].ptr, f0), ba[j]);
      if (full && bvec) MemC<32>::ld(addr<ESZ>(d.t[2].ptr, f0), bb[j]);
#pragma unroll
      for (int e = 0; e < V; ++e) {
        const bool in = vj[j] < vend && f0 + (IDX)e < d.nelem;
        if (in && !(full && avec)) MemC<ESZ>::ld(addr<ESZ>(d.t[1].ptr, off[1]), ba[j] + e * EW);
        if (in && !(full && bvec)) MemC<ESZ>::ld(addr<ESZ>(d.t[2].ptr, off[2]), bb[j] + e * EW);
        coff[j][e] = off[0];
        odo_inc1<D, 3, false, IDX>(d, u, off, oob);
      }
      odo_step<D, 3, false, IDX>(d, u, off, oob);
    }
#pragma unroll
    for (int j = 0; j < K; ++j) {
      if (vj[j] >= vend) continue;
      const IDX f0 = vj[j] * (IDX)V;
      uint32_t r[NW];
#pragma unroll
      for (int e = 0; e < V; ++e)
        Elem<ESZ>::put(r + e * EW,
                       bop<OP>(Elem<ESZ>::get(ba[j] + e * EW), Elem<ESZ>::get(bb[j] + e * EW)));
      if (cvec && f0 + (IDX)V <= d.nelem) {
        Mem<32>::st((void*)addr<ESZ>(d.t[0].ptr, f0), r);
      } else {
#pragma unroll
        for (int e = 0; e < V; ++e)
          if (f0 + (IDX)e < d.nelem)
            Mem<ESZ>::st((void*)addr<ESZ>(d.t[0].ptr, coff[j][e]), r + e * EW);
      }
    }
  }
}

// ------------------------------------------------------------------ row windows (short odd rows)
// When the innermost extent n is odd and short (3, 5, 7, ... up to 31 for embed, 64 for binary),
// or the output is not dense-and-aligned (a view, a misaligned base; rows up to 4096), a vector
// is one counter row.  A warp takes a group of W windows of 32 rows (W = d.rwin = ceil(16 / n)
// <= 8, so a group holds >= 16 elements per lane): lane i steps the odometer over rows b + i,
// b + 32 + i, ... (Alg 2 once, then the carry deltas) and parks each row's offsets in the
// warp's shared-memory row table.
// The warp then sweeps the group's rows * n elements lane by lane: element e = 32 j + lane
// lies in row r = e / n (one multiply-high by the plan's magic rmag, exact while e n < 2^32) and
// column e - r n.  The table holds each tensor's offset rebased to the element index,
// off'(r) = off(r) - r n tau, so element e sits at off'(r) + e tau, and (embed) the bound
// lim(r) = r n + m (0 when the row is out of src bounds), so "column < m" is e < lim(r).
// Consecutive lanes touch consecutive elements of every row-contiguous tensor, so accesses
// coalesce at any alignment and no lane branches on a row end; a tensor dense in the counter
// (dst, c) is addressed at the group base + e.  K elements per lane are loaded before any is
// stored.  In stride decomposition (tuning only) groups are single windows.
constexpr int kRowsWinMax = 8;                    // windows per group (plan: rwin <= this)
constexpr int kRowsTab = 32 * kRowsWinMax;        // row-table entries per warp

template <typename IDX>
struct alignas(2 * sizeof(IDX)) RowSrc {
  IDX off;   // rebased src offset
  IDX lim;   // element bound: e < lim <=> the element's column reads src
};

template <int ESZ, typename IDX, int K, bool DD, bool T1>
__device__ __forceinline__ void embed_rows_group(const Desc<IDX>& d, IDX gbase, uint32_t tot,
                                                 const RowSrc<IDX>* ts, const IDX* td, int lane) {
  constexpr int EW = ESZ / 4;
  const uint32_t mg = d.rmag;
  const IDX tau0 = T1 ? IDX(1) : d.t[0].tau, tau1 = T1 ? IDX(1) : d.t[1].tau;
  const char* src = (const char*)d.t[1].ptr;
  char* dst = (char*)d.t[0].ptr;
  for (uint32_t e0 = 0; e0 < tot; e0 += 32 * K) {
    uint32_t buf[K][EW];
    IDX doff[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const uint32_t e = e0 + 32u * j + (uint32_t)lane;
      const uint32_t r = min(__umulhi(e, mg), (uint32_t)kRowsTab - 1u);  // past tot: any entry
      const RowSrc<IDX> rs = ts[r];
      if (!DD) doff[j] = td[r] + (IDX)e * tau0;
      Mem<ESZ>::ld_or0(src + (uint64_t)(rs.off + (IDX)e * tau1) * ESZ, (IDX)e < rs.lim, buf[j]);
    }
    char* p = dst + (uint64_t)(gbase + (IDX)e0 + (IDX)lane) * ESZ;
#pragma unroll
    for (int j = 0; j < K; ++j)
      if (e0 + 32u * j + (uint32_t)lane < tot)
        Mem<ESZ>::st(DD ? (void*)(p + 32 * ESZ * j) : (void*)(dst + (uint64_t)doff[j] * ESZ),
                     buf[j]);
  }
}

// Long rows (plan rwarp): a whole warp sweeps one row at a time -- lane i takes
// columns i, i + 32, ... of that row, whose offsets and bound are uniform across the warp -- so
// there is no per-element table lookup; KW columns per lane are loaded before any is stored.
template <int ESZ, typename IDX, int KW, bool T1>
__device__ __forceinline__ void embed_warp_row(const Desc<IDX>& d, IDX so, IDX dof, IDX mrow,
                                               IDX n, int lane) {
  constexpr int EW = ESZ / 4;
  const IDX tau0 = T1 ? IDX(1) : d.t[0].tau, tau1 = T1 ? IDX(1) : d.t[1].tau;
  const char* sp = (const char*)d.t[1].ptr + (uint64_t)so * ESZ;
  char* dp = (char*)d.t[0].ptr + (uint64_t)dof * ESZ;
  for (IDX c0 = (IDX)lane; c0 < n; c0 += 32 * KW) {
    uint32_t buf[KW][EW];
#pragma unroll
    for (int j = 0; j < KW; ++j) {
      const IDX c = c0 + (IDX)(32 * j);
#pragma unroll
      for (int q = 0; q < EW; ++q) buf[j][q] = 0u;
      if (c < mrow) Mem<ESZ>::ld(sp + (uint64_t)(c * tau1) * ESZ, buf[j]);
    }
#pragma unroll
    for (int j = 0; j < KW; ++j) {
      const IDX c = c0 + (IDX)(32 * j);
      if (c < n) Mem<ESZ>::st(dp + (uint64_t)(c * tau0) * ESZ, buf[j]);
    }
  }
}

// A long row whose src is 32-byte aligned and whose length is a multiple of V (rows of a view
// window at an odd offset, say): lanes move 32-byte vectors -- aligned loads, and stores
// shifted to the 32-byte grid when the dst row is not (store_shifted); two vectors per lane in
// flight.  Columns >= mrow read as +0.
template <int ESZ, typename IDX>
__device__ __forceinline__ void embed_warp_row_vec(const Desc<IDX>& d, IDX so, IDX dof, IDX mrow,
                                                   IDX n, int lane) {
  constexpr int V = 32 / ESZ;
  constexpr int EW = ESZ / 4;
  constexpr int KV = 2;
  const char* sp = (const char*)d.t[1].ptr + (uint64_t)so * ESZ;
  char* dp = (char*)d.t[0].ptr + (uint64_t)dof * ESZ;
  const int sw = (int)(((uintptr_t)dp & 31u) >> 2);
  const IDX nv = n / (IDX)V;
  for (IDX v0 = 0; v0 < nv; v0 += 32 * KV) {
    uint32_t w[KV][8];
#pragma unroll
    for (int j = 0; j < KV; ++j) {
      const IDX vi = v0 + (IDX)(32 * j + lane);
      const IDX c0 = vi * (IDX)V;
      if (vi < nv && c0 + (IDX)V <= mrow) {
        Mem<32>::ld(sp + (uint64_t)c0 * ESZ, w[j]);
      } else {
#pragma unroll
        for (int e = 0; e < V; ++e) {
          if (vi < nv && c0 + (IDX)e < mrow) {
            Mem<ESZ>::ld(sp + (uint64_t)(c0 + (IDX)e) * ESZ, w[j] + e * EW);
          } else {
#pragma unroll
            for (int q = 0; q < EW; ++q) w[j][e * EW + q] = 0u;
          }
        }
      }
    }
#pragma unroll
    for (int j = 0; j < KV; ++j) {
      const IDX vb = v0 + (IDX)(32 * j);
      if (vb >= nv) break;
      const int nvalid = (nv - vb) < (IDX)32 ? (int)(nv - vb) : 32;
      char* a0 = dp + (uint64_t)vb * 32;
      if (sw == 0) {
        if (lane < nvalid) Mem<32>::st(a0 + 32 * lane, w[j]);
      } else {
        store_shifted<ESZ>(a0, w[j], sw, lane, nvalid);
      }
    }
  }
}

template <int D, int ESZ, typename IDX, int K>
__global__ void __launch_bounds__(kBlock) embed_rows_kernel(const __grid_constant__ Desc<IDX> d) {
  constexpr int EW = ESZ / 4;
  __shared__ RowSrc<IDX> tsrc[kBlock / 32][kRowsTab];
  __shared__ IDX tdst[kBlock / 32][kRowsTab];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const IDX warp = (IDX)blockIdx.x * (kBlock / 32) + (IDX)wib;
  const IDX base0 = warp * d.wmul;
  pdl_trigger();
  if (base0 >= d.nvec) return;
  const IDX vend = warp_end(d, base0);
  IDX u[D], off[2];
  uint32_t oob;
  odo_start<D, 2, true, IDX, true>(d, base0 + (IDX)lane, u, off, oob);
  const IDX n = (IDX)d.rowlen, m = d.scols;
  const IDX tau0 = d.t[0].tau, tau1 = d.t[1].tau;
  const bool ddense = d.t[0].vec != 0;
  const bool t1 = tau0 == IDX(1) && tau1 == IDX(1);  // both rows contiguous
  const int W = d.dv == (IDX)32 ? (int)d.rwin : 1;
  RowSrc<IDX>* ts = tsrc[wib];
  IDX* td = tdst[wib];
  for (int i = lane; i < kRowsTab; i += 32) {  // entries no group fills read nothing
    ts[i].off = 0;
    ts[i].lim = 0;
    td[i] = 0;
  }
  pdl_wait();
  IDX b = base0;
  while (b < vend) {
    // fill the row table: W windows (fewer at the end of the warp's range)
    uint32_t rows = 0;
    bool any = false;
    const IDX gb = b * n;  // counter element of the group's first row
    for (int w = 0; w < W && b < vend; ++w, b += d.dv) {
      const uint32_t nr = (vend - b) < (IDX)32 ? (uint32_t)(vend - b) : 32u;
      const bool rd = (uint32_t)lane < nr && oob == 0;  // row reads src
      IDX mr = m;  // columns of this row read from src
      if (d.seglen) {  // a segment s of a split axis: clamp(segm - s n, 0, n)
        const IDX s0 = u[D - 1] * n;
        mr = d.segm > s0 ? (d.segm - s0 < n ? d.segm - s0 : n) : IDX(0);
      }
      any = any || (rd && mr != 0);
      const IDX r0 = (IDX)(32 * w + lane) * n;  // group element index of the row's first element
      ts[32 * w + lane].off = off[1] - r0 * tau1;
      ts[32 * w + lane].lim = rd ? r0 + mr : IDX(0);
      td[32 * w + lane] = off[0] - r0 * tau0;
      rows = 32u * (uint32_t)w + nr;
      odo_step<D, 2, true, IDX, true>(d, u, off, oob);
    }
    __syncwarp();
    const uint32_t tot = rows * (uint32_t)n;
    if (ddense) {
      if (!__any_sync(0xffffffffu, any)) {
        // every row of the group is out of src bounds: a plain zero stream
        uint32_t z[EW];
#pragma unroll
        for (int q = 0; q < EW; ++q) z[q] = 0u;
        for (uint32_t e = lane; e < tot; e += 32)
          Mem<ESZ>::st((void*)addr<ESZ>(d.t[0].ptr, gb + (IDX)e), z);
      } else if (t1) {
        embed_rows_group<ESZ, IDX, K, true, true>(d, gb, tot, ts, td, lane);
      } else {
        embed_rows_group<ESZ, IDX, K, true, false>(d, gb, tot, ts, td, lane);
      }
    } else {
      embed_rows_group<ESZ, IDX, K, false, false>(d, gb, tot, ts, td, lane);
    }
    __syncwarp();
  }
}

// One group of the binary op: a and b offsets from the table, c dense (CD) or from the table.
template <int ESZ, typename IDX, int K, int OP, bool CD, bool T1>
__device__ __forceinline__ void binary_rows_group(const Desc<IDX>& d, IDX gbase, uint32_t tot,
                                                  const IDX* tc, const RowSrc<IDX>* tab,
                                                  int lane) {
  constexpr int EW = ESZ / 4;
  const uint32_t mg = d.rmag;
  const IDX sc = T1 ? IDX(1) : d.t[0].tau, sa = T1 ? IDX(1) : d.t[1].tau;
  const IDX sb = T1 ? IDX(1) : d.t[2].tau;
  char* c = (char*)d.t[0].ptr;
  const char* pa = (const char*)d.t[1].ptr;
  const char* pb = (const char*)d.t[2].ptr;
  for (uint32_t e0 = 0; e0 < tot; e0 += 32 * K) {
    uint32_t ba[K][EW], bb[K][EW];
    IDX coff[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const uint32_t e = e0 + 32u * j + (uint32_t)lane;
      const uint32_t r = min(__umulhi(e, mg), (uint32_t)kRowsTab - 1u);
      const RowSrc<IDX> ab = tab[r];  // .off = a, .lim = b (rebased offsets)
      if (!CD) coff[j] = tc[r] + (IDX)e * sc;
      MemC<ESZ>::ld_or0(pa + (uint64_t)(ab.off + (IDX)e * sa) * ESZ, e < tot, ba[j]);
      MemC<ESZ>::ld_or0(pb + (uint64_t)(ab.lim + (IDX)e * sb) * ESZ, e < tot, bb[j]);
    }
    char* p = c + (uint64_t)(gbase + (IDX)e0 + (IDX)lane) * ESZ;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      if (e0 + 32u * j + (uint32_t)lane >= tot) continue;
      uint32_t r[EW];
      Elem<ESZ>::put(r, bop<OP>(Elem<ESZ>::get(ba[j]), Elem<ESZ>::get(bb[j])));
      Mem<ESZ>::st(CD ? (void*)(p + 32 * ESZ * j) : (void*)(c + (uint64_t)coff[j] * ESZ), r);
    }
  }
}

template <int ESZ, typename IDX, int KW, int OP, bool T1>
__device__ __forceinline__ void binary_warp_row(const Desc<IDX>& d, IDX oc, IDX oa, IDX ob, IDX n,
                                                int lane) {
  constexpr int EW = ESZ / 4;
  const IDX sc = T1 ? IDX(1) : d.t[0].tau, sa = T1 ? IDX(1) : d.t[1].tau;
  const IDX sb = T1 ? IDX(1) : d.t[2].tau;
  char* cp = (char*)d.t[0].ptr + (uint64_t)oc * ESZ;
  const char* ap = (const char*)d.t[1].ptr + (uint64_t)oa * ESZ;
  const char* bp = (const char*)d.t[2].ptr + (uint64_t)ob * ESZ;
  for (IDX c0 = (IDX)lane; c0 < n; c0 += 32 * KW) {
    uint32_t ba[KW][EW], bb[KW][EW];
#pragma unroll
    for (int j = 0; j < KW; ++j) {
      const IDX c = c0 + (IDX)(32 * j);
      if (c < n) {
        MemC<ESZ>::ld(ap + (uint64_t)(c * sa) * ESZ, ba[j]);
        MemC<ESZ>::ld(bp + (uint64_t)(c * sb) * ESZ, bb[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < KW; ++j) {
      const IDX c = c0 + (IDX)(32 * j);
      if (c >= n) continue;
      uint32_t r[EW];
      Elem<ESZ>::put(r, bop<OP>(Elem<ESZ>::get(ba[j]), Elem<ESZ>::get(bb[j])));
      Mem<ESZ>::st(cp + (uint64_t)(c * sc) * ESZ, r);
    }
  }
}

template <int D, int ESZ, typename IDX, int K, int OP>
__global__ void __launch_bounds__(kBlock) binary_rows_kernel(const __grid_constant__ Desc<IDX> d) {
  __shared__ RowSrc<IDX> tab[kBlock / 32][kRowsTab];
  __shared__ IDX tcs[kBlock / 32][kRowsTab];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const IDX warp = (IDX)blockIdx.x * (kBlock / 32) + (IDX)wib;
  const IDX base0 = warp * d.wmul;
  pdl_trigger();
  if (base0 >= d.nvec) return;
  const IDX vend = warp_end(d, base0);
  IDX u[D], off[3];
  uint32_t oob;
  odo_start<D, 3, false, IDX>(d, base0 + (IDX)lane, u, off, oob);
  const IDX n = (IDX)d.rowlen;
  const IDX sc = d.t[0].tau, sa = d.t[1].tau, sb = d.t[2].tau;
  const bool cd = d.t[0].vec != 0;
  const bool t1 = sc == IDX(1) && sa == IDX(1) && sb == IDX(1);
  const int W = d.dv == (IDX)32 ? (int)d.rwin : 1;
  pdl_wait();
  IDX b = base0;
  while (b < vend) {
    uint32_t rows = 0;
    const IDX gb = b * n;
    for (int w = 0; w < W && b < vend; ++w, b += d.dv) {
      const uint32_t nr = (vend - b) < (IDX)32 ? (uint32_t)(vend - b) : 32u;
      const IDX r0 = (IDX)(32 * w + lane) * n;
      tab[wib][32 * w + lane].off = off[1] - r0 * sa;
      tab[wib][32 * w + lane].lim = off[2] - r0 * sb;
      tcs[wib][32 * w + lane] = off[0] - r0 * sc;
      rows = 32u * (uint32_t)w + nr;
      odo_step<D, 3, false, IDX>(d, u, off, oob);
    }
    __syncwarp();
    if (cd && t1)
      binary_rows_group<ESZ, IDX, K, OP, true, true>(d, gb, rows * (uint32_t)n, tcs[wib],
                                                     tab[wib], lane);
    else if (cd)
      binary_rows_group<ESZ, IDX, K, OP, true, false>(d, gb, rows * (uint32_t)n, tcs[wib],
                                                      tab[wib], lane);
    else
      binary_rows_group<ESZ, IDX, K, OP, false, false>(d, gb, rows * (uint32_t)n, tcs[wib],
                                                       tab[wib], lane);
    __syncwarp();
  }
}

// Row windows, warp per row (long rows, plan rwarp): the lane-per-row odometer of the row-window
// kernels, then the warp sweeps each of its 32 rows in turn with uniform offsets and bound.
template <int D, int ESZ, typename IDX>
__global__ void __launch_bounds__(kBlock) embed_rowsw_kernel(const __grid_constant__ Desc<IDX> d) {
  const int lane = threadIdx.x & 31;
  const IDX warp = (IDX)blockIdx.x * (kBlock / 32) + (IDX)(threadIdx.x >> 5);
  const IDX base0 = warp * d.wmul;
  pdl_trigger();
  if (base0 >= d.nvec) return;
  const IDX vend = warp_end(d, base0);
  IDX u[D], off[2];
  uint32_t oob;
  odo_start<D, 2, true, IDX, true>(d, base0 + (IDX)lane, u, off, oob);
  const IDX n = (IDX)d.rowlen, m = d.scols;
  const bool t1 = d.t[0].tau == IDX(1) && d.t[1].tau == IDX(1);
  constexpr int KW = 64 / ESZ;  // 64 B of loads per lane in flight
  pdl_wait();
  for (IDX b = base0; b < vend; b += d.dv) {
    const uint32_t nr = (vend - b) < (IDX)32 ? (uint32_t)(vend - b) : 32u;
    IDX mr = m;  // columns of the lane's row read from src
    if (d.seglen) {
      const IDX s0 = u[D - 1] * n;
      mr = d.segm > s0 ? (d.segm - s0 < n ? d.segm - s0 : n) : IDX(0);
    }
    if (oob != 0) mr = 0;
    for (uint32_t i = 0; i < nr; ++i) {
      const IDX so = shfl_idx(off[1], (int)i), dof = shfl_idx(off[0], (int)i);
      const IDX mrow = shfl_idx(mr, (int)i);
      const bool vec_ok = t1 && n % (IDX)(32 / ESZ) == 0 &&
                          (((uintptr_t)d.t[1].ptr + (uint64_t)so * ESZ) & 31u) == 0 &&
                          (((uintptr_t)d.t[0].ptr + (uint64_t)dof * ESZ) & (ESZ - 1)) == 0;
      if (vec_ok)
        embed_warp_row_vec<ESZ, IDX>(d, so, dof, mrow, n, lane);
      else if (t1)
        embed_warp_row<ESZ, IDX, KW, true>(d, so, dof, mrow, n, lane);
      else
        embed_warp_row<ESZ, IDX, KW, false>(d, so, dof, mrow, n, lane);
    }
    odo_step<D, 2, true, IDX, true>(d, u, off, oob);
  }
}

template <int D, int ESZ, typename IDX, int OP>
__global__ void __launch_bounds__(kBlock) binary_rowsw_kernel(const __grid_constant__ Desc<IDX> d) {
  const int lane = threadIdx.x & 31;
  const IDX warp = (IDX)blockIdx.x * (kBlock / 32) + (IDX)(threadIdx.x >> 5);
  const IDX base0 = warp * d.wmul;
  pdl_trigger();
  if (base0 >= d.nvec) return;
  const IDX vend = warp_end(d, base0);
  IDX u[D], off[3];
  uint32_t oob;
  odo_start<D, 3, false, IDX>(d, base0 + (IDX)lane, u, off, oob);
  const IDX n = (IDX)d.rowlen;
  const bool t1 = d.t[0].tau == IDX(1) && d.t[1].tau == IDX(1) && d.t[2].tau == IDX(1);
  constexpr int KW = 32 / ESZ;  // two operands: 64 B of loads per lane in flight
  pdl_wait();
  for (IDX b = base0; b < vend; b += d.dv) {
    const uint32_t nr = (vend - b) < (IDX)32 ? (uint32_t)(vend - b) : 32u;
    for (uint32_t i = 0; i < nr; ++i) {
      const IDX oc = shfl_idx(off[0], (int)i), oa = shfl_idx(off[1], (int)i);
      const IDX ob = shfl_idx(off[2], (int)i);
      if (t1)
        binary_warp_row<ESZ, IDX, KW, OP, true>(d, oc, oa, ob, n, lane);
      else
        binary_warp_row<ESZ, IDX, KW, OP, false>(d, oc, oa, ob, n, lane);
    }
    odo_step<D, 3, false, IDX>(d, u, off, oob);
  }
}

// ------------------------------------------------------------------ expected value
// m_k = sum_t t_k p[t] (Alg 11) in fp64.  p is the counter tensor itself (dense,
// never merged), so vector v starts at element v*V: the loads need no odometer.  Two kernels:
// ev_tma_kernel (the fast path: p streamed by TMA bulk copies into a ring of shared-memory
// stages, one persistent block per SM) and ev_kernel (batched 32-byte loads; any alignment or
// vector width).  The digits (the weights t_k) advance with the Alg 3 odometer as vectors are
// consumed.  Per
// vector the outer digits are constant, so with s = sum_e p_e:  acc_k += u_k * s, and the
// vector digit contributes (first row/col) * s plus the in-vector weights.  Per-lane fp64
// accumulators, then a fixed-order warp butterfly, a fixed-order cross-warp sum, one partial per
// block, and the last block (ticket) sums the partials in a fixed order: deterministic run to
// run ("each thread computes its own pre-result and these pre-results are amalgamated").

// ---- expected-value accumulation with deferred weights
// For one lane, sum_v u_k(v) s(v) (s = mass of vector v) telescopes to
//     u_k(final) * S  -  sum over changes of digit k of (new - old) * S_at_change
// where S is the running mass.  So per vector only S += s (plus the in-vector weights) is
// computed, and digit k costs one FMA when it changes -- which the odometer makes amortised
// O(1) per step, the same argument as Alg 3's.  Exact for integer-valued inputs; for
// real inputs the extra rounding is a few ulps of sum |t_k p| (DESIGN.md §EV numerics).
template <int D>
struct EvAcc {
  double S;        // running mass
  double Wr, Wc;   // in-vector row / column weighted mass
  double ev[D];    // -sum (delta u_k) * S_at_change
};

template <int D, typename IDX>
__device__ __forceinline__ void ev_acc_init(EvAcc<D>& a) {
  a.S = a.Wr = a.Wc = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) a.ev[k] = 0.0;
}

// The odometer on digits only (no tensor offsets), recording weight events.
template <int D, typename IDX>
__device__ __forceinline__ void digits_step_ev(const Desc<IDX>& d, IDX (&u)[D], EvAcc<D>& a) {
  bool carry = false;
#pragma unroll
  for (int k = D - 1; k >= 0; --k) {
    if (k > d.khi) continue;
    const IDX old = u[k];
    IDX nu = old + d.dlt[k] + (carry ? IDX(1) : IDX(0));
    carry = nu >= d.ext[k];
    if (carry) nu -= d.ext[k];
    u[k] = nu;
    if (nu != old) {  // one exact conversion of the signed change (|delta| < 2^53)
      const double delta = (double)((int64_t)nu - (int64_t)old);
      a.ev[k] = fma(-delta, a.S, a.ev[k]);
    }
    if (k <= d.klo && !carry) break;
  }
}

template <int ESZ, int V, typename IDX>
__device__ __forceinline__ void ev_load(const TensorAcc<IDX>& t, IDX v, uint32_t* w) {
  constexpr int EW = ESZ / 4;
  const IDX off = v * (IDX)V;
  if (V > 1 && t.vec) {
    Mem<V * ESZ>::ld(addr<ESZ>(t.ptr, off), w);
  } else {
#pragma unroll
    for (int e = 0; e < V; ++e) Mem<ESZ>::ld(addr<ESZ>(t.ptr, off + (IDX)e), w + e * EW);
  }
}

template <int D, typename IDX>
__device__ __forceinline__ void ev_decode(const Desc<IDX>& d, IDX v, IDX (&u)[D]) {
  decode_digits<D, IDX>(d, v, u);
}

// in-vector row / column weighted sums of a collapsed vector with a compile-time row length
template <int V, int LGL>
__device__ __forceinline__ void ev_collapsed_weights(const double (&x)[V], double& wr, double& wc) {
#pragma unroll
  for (int e = 1; e < V; ++e) {
    constexpr int L = 1 << LGL;
    const int r = e / L, c = e % L;
    if (r) wr = fma((double)r, x[e], wr);
    if (c) wc = fma((double)c, x[e], wc);
  }
}

// One vector: S += sum_e p_e; the in-vector row (e >> lgL) and column (e & (L-1)) weights
// accumulate into Wr / Wc.  lgL is a runtime value but e is unrolled.
template <int D, int ESZ, int V, typename IDX>
__device__ __forceinline__ void ev_accumulate(const Desc<IDX>& d, const uint32_t* w,
                                              EvAcc<D>& a) {
  constexpr int EW = ESZ / 4;
  const uint32_t lgL = d.lgL;
  double x[V];
#pragma unroll
  for (int e = 0; e < V; ++e) x[e] = (double)Elem<ESZ>::get(w + e * EW);
  double sum = x[0];
#pragma unroll
  for (int e = 1; e < V; ++e) sum += x[e];
  a.S += sum;
  if (V > 1 && d.collapsed == 0) {
    // one row per vector (lgL = log2 V): column weight e, row weight 0 -- immediate constants,
    // the same FMA sequence as the general path below
    double wc = 0.0;
#pragma unroll
    for (int e = 1; e < V; ++e) wc = fma((double)e, x[e], wc);
    a.Wc += wc;
  } else if (V > 1) {
    // rows shorter than a vector (2 or 4 elements): the row / column of element e from lgL.
    // The usual row lengths get immediate weights (warp-uniform branch); the generic form
    // converts two integers per element ((8192,8192,4) f32, 268 MB: 3.97 -> 5.35 TB/s).
    double wr = 0.0, wc = 0.0;
    if (lgL == 2 && V >= 8) {
      ev_collapsed_weights<V, 2>(x, wr, wc);
    } else if (lgL == 1 && V >= 4) {
      ev_collapsed_weights<V, 1>(x, wr, wc);
    } else {
#pragma unroll
      for (int e = 1; e < V; ++e) {
        const uint32_t r = (uint32_t)e >> lgL, c = (uint32_t)e & ((1u << lgL) - 1u);
        if (r) wr = fma((double)r, x[e], wr);
        if (c) wc = fma((double)c, x[e], wc);
      }
    }
    a.Wr += wr;
    a.Wc += wc;
  }
}

// Weight slots of one lane at the end: slot k < D-1 -> u_k S + ev_k; slot D-1 (the vector digit)
// -> vmul (u S + ev) + (Wr if collapsed else Wc); slot D (collapsed column) -> Wc; slot D+1 ->
// the mass S.
template <int D, typename IDX>
__device__ __forceinline__ void ev_finish(const Desc<IDX>& d, const IDX (&u)[D],
                                          const EvAcc<D>& a, double (&acc)[D + 2]) {
#pragma unroll
  for (int k = 0; k < D - 1; ++k) acc[k] = fma((double)u[k], a.S, a.ev[k]);
  const double vmul = (double)(d.rowmul + d.colmul);
  const bool coll = d.collapsed != 0;
  acc[D - 1] = fma(vmul, fma((double)u[D - 1], a.S, a.ev[D - 1]), coll ? a.Wr : a.Wc);
  acc[D] = coll ? a.Wc : 0.0;
  acc[D + 1] = a.S;  // the mass (slab-sharded EV amalgamation term)
}

// partial slots per block, padded to a power of two so the final sum reads them coalesced
__host__ __device__ constexpr int ev_slot_pad(int ns) {
  return ns <= 1 ? 1 : ns <= 2 ? 2 : ns <= 4 ? 4 : ns <= 8 ? 8 : ns <= 16 ? 16 : 32;
}

// Warp reduce-scatter of NS partial sums (fixed order): at each butterfly level a lane keeps
// half of its slots and adds the partner's copy of them, so after log2(P) levels (P = NS rounded
// up to a power of two) every lane holds one slot's sum over its group and plain butterfly levels
// finish it -- NS + log2 levels of shuffles instead of 5 * NS.  Returns the value; `slot` gets
// its slot index (lanes with the same slot hold identical values).
template <int NS>
__device__ __forceinline__ double warp_reduce_scatter(const double (&acc)[NS], int lane,
                                                      int& slot) {
  constexpr int P = NS <= 1 ? 1 : NS <= 2 ? 2 : NS <= 4 ? 4 : NS <= 8 ? 8 : NS <= 16 ? 16 : 32;
  double a[P];
#pragma unroll
  for (int k = 0; k < P; ++k) a[k] = k < NS ? acc[k] : 0.0;
  int base = 0;
#pragma unroll
  for (int L = 0; L < 5; ++L) {
    const int o = 16 >> L;
    const int h = P >> L;
    if (h > 1) {
      const int half = h / 2;
      const bool up = (lane & o) != 0;
#pragma unroll
      for (int j = 0; j < half; ++j) {
        const double send = up ? a[j] : a[j + half];
        const double keep = up ? a[j + half] : a[j];
        a[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
      if (up) base += half;
    } else {
      a[0] += __shfl_xor_sync(0xffffffffu, a[0], o);
    }
  }
  slot = base;
  return a[0];
}

// 32-byte chunks per thread in flight in the final ordered sum, and the poll's sleep (ns)
// (6 x 256 threads x 4 doubles cover the 592 x 8 partials of a d <= 6 expected value at 4 blocks
// per SM in ONE round of loads: C3 back to back 24.94 -> 24.56 us against 4 chunks, which took
// a second round trip for the last 160 chunks; profiles/r02_ev18_final_chunks*)
#ifndef TRIOT_EV_FINAL_CHUNKS
#define TRIOT_EV_FINAL_CHUNKS 6
#endif
#ifndef TRIOT_EV_POLL_SLEEP
#define TRIOT_EV_POLL_SLEEP 64
#endif

// Ordered sum of `nparts` partials laid out [part][P slots] (P = ev_slot_pad(NS)), read as
// 32-byte chunks, 4 chunks per thread in flight: chunk c holds the doubles 4c .. 4c+3, i.e. slots
// (4c + q) % P, and since BLOCK * 4 is a multiple of P thread t always meets slots (4t + q) % P.
// Lanes that meet the same slots are combined by a butterfly, warps in index order: a fixed
// function of the partials, whichever block runs it.  Leaves the NS totals in sm[0][0..NS-1].
template <int NS, int BLOCK, int CH = TRIOT_EV_FINAL_CHUNKS>
__device__ __forceinline__ void ordered_slot_sum(const double* src, unsigned nparts,
                                                 double (&sm)[BLOCK / 32][NS]) {
  constexpr int P = ev_slot_pad(NS);
  static_assert((4 * BLOCK) % P == 0, "slots must tile the block");
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const unsigned total = nparts * (unsigned)P;
  const unsigned nchunk = (total + 3u) / 4u;
  double f[4] = {0.0, 0.0, 0.0, 0.0};
  for (unsigned c0 = threadIdx.x; c0 < nchunk; c0 += (unsigned)CH * BLOCK) {
    uint32_t w[CH][8];
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      const unsigned c = c0 + (unsigned)i * BLOCK;
      if (c < nchunk && 4u * c + 3u < total) {
        asm volatile("ld.global.cg.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(w[i][0]), "=r"(w[i][1]), "=r"(w[i][2]), "=r"(w[i][3]), "=r"(w[i][4]),
                       "=r"(w[i][5]), "=r"(w[i][6]), "=r"(w[i][7])
                     : "l"(src + 4 * (size_t)c));
      } else {  // past the end, or a ragged last chunk (P < 4): element by element
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double x = (c < nchunk && 4u * c + q < total) ? __ldcg(src + 4 * (size_t)c + q) : 0.0;
          w[i][2 * q] = (uint32_t)__double2loint(x);
          w[i][2 * q + 1] = (uint32_t)__double2hiint(x);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < CH; ++i)
#pragma unroll
      for (int q = 0; q < 4; ++q) f[q] += __hiloint2double((int)w[i][2 * q + 1], (int)w[i][2 * q]);
  }
  if (P >= 4) {
    constexpr int OMIN = P >= 4 ? P / 4 : 1;
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int o = 16; o >= OMIN; o >>= 1) f[q] += __shfl_xor_sync(0xffffffffu, f[q], o);
    if (lane < OMIN) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (4 * lane + q < NS) sm[wib][4 * lane + q] = f[q];
    }
  } else {
    double g[2] = {0.0, 0.0};
#pragma unroll
    for (int q = 0; q < 4; ++q) g[q % (P < 1 ? 1 : P)] += f[q];
#pragma unroll
    for (int q = 0; q < (P < 1 ? 1 : P); ++q) {
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) g[q] += __shfl_xor_sync(0xffffffffu, g[q], o);
      if (lane == 0 && q < NS) sm[wib][q] = g[q];
    }
  }
  __syncthreads();
  if (threadIdx.x < NS) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < BLOCK / 32; ++w) t += sm[w][threadIdx.x];
    sm[0][threadIdx.x] = t;  // each thread reads and writes its own column only
  }
  __syncthreads();
}

// out[j] from the slot totals in sm[0][]; a block of a larger PMF adds offset * mass
template <int NS, int BLOCK, typename IDX>
__device__ __forceinline__ void ev_write_out(const Desc<IDX>& d,
                                             const double (&sm)[BLOCK / 32][NS]) {
  if (threadIdx.x < (unsigned)d.d_out) {
    const int sl = d.slot_of_axis[threadIdx.x];
    double v = sl >= 0 ? sm[0][sl] : 0.0;
    // sum_t (off_j + t_j) p[t] = m_j + off_j * mass (one rounding)
    if ((int)threadIdx.x < d.nax && d.offd[threadIdx.x] != 0.0)
      v = fma(d.offd[threadIdx.x], sm[0][d.slot_of_axis[d.nax]], v);
    ((double*)d.out)[threadIdx.x] = v;
  }
}

// Fixed-order block reduction ("each thread computes its own pre-result and these pre-results
// are amalgamated"): warp reduce-scatter, warps in index order -> one partial per block
// (slot blockIdx); then every block but the last-launched one *arrives* on a counter with a
// release reduction and exits -- no block waits on an atomic's reply (a ticket per block held
// its slot for ~0.5-1 us: profiles/r02_ev4_tail.jsonl, r02_ev7_k*) -- while the last-launched
// block (dispatched last, so every other block is resident or done) has one thread poll the
// counter until the grid - 1 arrivals are in, then sums the partials in block order
// (ordered_slot_sum) and writes the result.  Deterministic for a fixed grid; the counter is left
// at 0 for the next call.  (Measured alternatives: profiles/r02_ev*.)
template <int NS, int BLOCK, typename IDX>
__device__ __forceinline__ void ev_reduce(const Desc<IDX>& d, double (&acc)[NS]) {
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  constexpr int GRP = NS <= 1 ? 32 : NS <= 2 ? 16 : NS <= 4 ? 8 : NS <= 8 ? 4 : NS <= 16 ? 2 : 1;
  __shared__ double sm[BLOCK / 32][NS];
  {
    int slot;
    const double v = warp_reduce_scatter<NS>(acc, lane, slot);
    if ((lane & (GRP - 1)) == 0 && slot < NS) sm[wib][slot] = v;
  }
  __syncthreads();
  if (gridDim.x == 1 && !d.split) {
    // a single block (a small PMF: launch_geometry): its slot sums are the totals -- no partial
    // in global memory, no counter, no L2 round trips (a 128-byte EV in a CUDA graph: 2.30 ->
    // 1.31 us per op).  The same values as the general path gives for one block.
    if (threadIdx.x < NS) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < BLOCK / 32; ++w) t += sm[w][threadIdx.x];
      sm[0][threadIdx.x] = t;  // each thread reads and writes its own column only
    }
    __syncthreads();
    ev_write_out<NS, BLOCK, IDX>(d, sm);
    return;
  }
  if (d.cluster > 1 && !d.split) {
    // The grid is one thread-block cluster (a mid-size PMF: launch_geometry).  Every block
    // stores its slot sums into block 0's shared memory (distributed shared memory) and
    // arrives on the cluster barrier with release; block 0 waits with acquire, adds the
    // partials in block order and writes the result: the same fixed order as the general
    // path, with no partial in global memory, no counter and no L2 round trip.
    __shared__ double cl[TRIOT_CLUSTER_MAX][NS];
    unsigned rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    if (threadIdx.x < NS) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < BLOCK / 32; ++w) t += sm[w][threadIdx.x];
      uint32_t remote;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                   : "=r"(remote)
                   : "r"((uint32_t)__cvta_generic_to_shared(&cl[rank][threadIdx.x])), "r"(0u));
      asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(remote), "d"(t) : "memory");
    }
    asm volatile("barrier.cluster.arrive.release;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire;" ::: "memory");
    if (rank != 0) return;
    if (threadIdx.x < NS) {
      double t = 0.0;
      for (unsigned r = 0; r < d.cluster; ++r) t += cl[r][threadIdx.x];
      sm[0][threadIdx.x] = t;
    }
    __syncthreads();
    ev_write_out<NS, BLOCK, IDX>(d, sm);
    return;
  }
  unsigned* ctr = (unsigned*)d.ws;
  double* part = (double*)((char*)d.ws + TRIOT_EV_WS_HEADER);
  constexpr int P = ev_slot_pad(NS);
  static_assert(BLOCK % P == 0, "slots must tile the block");
  if (threadIdx.x < P) {  // the block-order sum of slot t over the warps (padding slots: +0.0)
    double t = 0.0;
    if (threadIdx.x < NS) {
#pragma unroll
      for (int w = 0; w < BLOCK / 32; ++w) t += sm[w][threadIdx.x];
    }
    part[(size_t)blockIdx.x * P + threadIdx.x] = t;
  }
  if (d.split) return;  // ev_final_kernel sums the partials once this grid has completed
  __syncthreads();      // this block's partial stores precede thread 0's release below
  if (blockIdx.x != gridDim.x - 1) {
    if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    TRIOT_TRACE(3);
    return;
  }
  if (threadIdx.x == 0) {
    const unsigned target = gridDim.x - 1;
    unsigned c;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(c) : "l"(ctr) : "memory");
    while (c < target) {
#if TRIOT_EV_POLL_SLEEP
      __nanosleep(TRIOT_EV_POLL_SLEEP);
#endif
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(c) : "l"(ctr) : "memory");
    }
    // synchronizes with every arrival's release (they form a release sequence on the counter)
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(c) : "l"(ctr) : "memory");
    *ctr = 0u;  // every arrival is in: leave the counter ready for the next call
  }
  __syncthreads();  // the acquire (thread 0) orders every thread's partial loads below
  TRIOT_TRACE(5);
  ordered_slot_sum<NS, BLOCK>(part, gridDim.x, sm);
  TRIOT_TRACE(6);
  ev_write_out<NS, BLOCK, IDX>(d, sm);
}

// Amalgamation of pre-results: out[j] = sum_r rows[r][j], rows in order (fixed order:
// deterministic).  Sums the per-slab results of the host-streamed expected value and the
// per-rank results of the sharded one.
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) sum_rows_kernel(double* out, const double* rows,
                                                         uint64_t nrows, uint64_t ncols) {
  pdl_trigger();
  pdl_wait();
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= ncols) return;
  double t = 0.0;
  for (uint64_t r = 0; r < nrows; ++r) t += __ldcg(rows + r * ncols + j);
  out[j] = t;
}

// Second half of a split reduction: launched after the reduction kernel with programmatic
// stream serialization; griddepcontrol.wait returns once every partial is written and visible.
// Fixed order for a fixed partial count: per thread a strided sequential sum, warp butterfly,
// warps in index order -- deterministic like the single-kernel ticket path.
constexpr int kFinBlock = 512;
struct EvFin {
  const double* part;
  double* out;
  uint32_t nblk;
  int32_t ns, d_out;
  int32_t slot_of_axis[TRIOT_MAXD + 1];
  int32_t nax;
  double offd[TRIOT_MAXD];
};
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) ev_final_kernel(const __grid_constant__ EvFin f) {
  constexpr int NSMAX = TRIOT_MAXD + 2;
  pdl_trigger();
  pdl_wait();
  // same order as ev_reduce's last block: slot t % P, blocks in order, butterfly, warps
  const unsigned P = (unsigned)ev_slot_pad(f.ns);
  const unsigned total = f.nblk * P;
  double a = 0.0;
  for (unsigned i0 = threadIdx.x; i0 < total; i0 += 4 * BLOCK) {
    double x[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const unsigned idx = i0 + (unsigned)i * BLOCK;
      x[i] = idx < total ? __ldcg(f.part + idx) : 0.0;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) a += x[i];
  }
  __shared__ double sm[BLOCK / 32][NSMAX];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  for (unsigned o = 16; o >= P; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  if (lane < f.ns) sm[wib][lane] = a;
  __syncthreads();
  __shared__ double tot[NSMAX];
  if ((int)threadIdx.x < f.ns) {
    double t = 0.0;
    for (int w = 0; w < BLOCK / 32; ++w) t += sm[w][threadIdx.x];
    tot[threadIdx.x] = t;
  }
  __syncthreads();
  if ((int)threadIdx.x < f.d_out) {
    const int sl = f.slot_of_axis[threadIdx.x];
    double t = sl >= 0 ? tot[sl] : 0.0;
    if ((int)threadIdx.x < f.nax && f.offd[threadIdx.x] != 0.0)
      t = fma(f.offd[threadIdx.x], tot[f.slot_of_axis[f.nax]], t);
    f.out[threadIdx.x] = t;
  }
}

template <int D, int ESZ, int V, typename IDX, int K, int MINB = 4>
__global__ void __launch_bounds__(kBlock, MINB) ev_kernel(const __grid_constant__ Desc<IDX> d) {
  constexpr int EW = ESZ / 4;
  constexpr int NW = V * EW;
  constexpr int NS = D + 2;  // D digit slots + collapsed column slot + mass
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const IDX warp = (IDX)blockIdx.x * (kBlock / 32) + (IDX)wib;
  const IDX base0 = warp * d.wmul;
  double acc[NS];
#pragma unroll
  for (int k = 0; k < NS; ++k) acc[k] = 0.0;
  pdl_trigger();
  pdl_wait();
  TRIOT_TRACE(0);
  if (base0 < d.nvec) {
    const IDX vend = warp_end(d, base0);
    const IDX dv = d.dv;
    IDX v = base0 + (IDX)lane;
    IDX u[D];
    ev_decode<D, IDX>(d, v, u);
    EvAcc<D> a;
    ev_acc_init<D, IDX>(a);
    for (IDX b = base0; b < vend; b += (IDX)K * dv) {
      if (b == base0) TRIOT_TRACE(1);
      uint32_t buf[K][NW];
#pragma unroll
      for (int j = 0; j < K; ++j)
        if (v + (IDX)j * dv < vend) ev_load<ESZ, V, IDX>(d.t[0], v + (IDX)j * dv, buf[j]);
#pragma unroll
      for (int j = 0; j < K; ++j) {
        if (v < vend) ev_accumulate<D, ESZ, V, IDX>(d, buf[j], a);
        digits_step_ev<D, IDX>(d, u, a);
        v += dv;
      }
    }
    ev_finish<D, IDX>(d, u, a, acc);
  }
  TRIOT_TRACE(2);
  ev_reduce<NS, kBlock, IDX>(d, acc);
  TRIOT_TRACE(4);
}

// Expected value of a view (NEXT-1): as ev_kernel, but p is the window of a larger base, so
// each lane tracks p's offset with the odometer (Alg 2 at the start, per-step carry deltas after
// it).  Two copies of the digits: `uo` runs K steps ahead for the loads' offsets, `u` follows
// the accumulation and records the telescoped weight events.
template <int D, int ESZ, int V, typename IDX, int K>
__global__ void __launch_bounds__(kBlock, 4) ev_view_kernel(const __grid_constant__ Desc<IDX> d) {
  constexpr int EW = ESZ / 4;
  constexpr int NW = V * EW;
  constexpr int NS = D + 2;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const IDX warp = (IDX)blockIdx.x * (kBlock / 32) + (IDX)wib;
  const IDX base0 = warp * d.wmul;
  double acc[NS];
#pragma unroll
  for (int k = 0; k < NS; ++k) acc[k] = 0.0;
  pdl_trigger();
  pdl_wait();
  if (base0 < d.nvec) {
    const IDX vend = warp_end(d, base0);
    const IDX dv = d.dv;
    const uint32_t lgL = d.lgL;
    IDX v = base0 + (IDX)lane;
    IDX uo[D], off[1];
    uint32_t oob;
    odo_start<D, 1, false, IDX>(d, v, uo, off, oob);
    IDX u[D];
#pragma unroll
    for (int k = 0; k < D; ++k) u[k] = uo[k];
    EvAcc<D> a;
    ev_acc_init<D, IDX>(a);
    for (IDX b = base0; b < vend; b += (IDX)K * dv) {
      uint32_t buf[K][NW];
      IDX offj[K], colj[K];
#pragma unroll
      for (int j = 0; j < K; ++j) {
        offj[j] = off[0];
        colj[j] = uo[D - 1] * (IDX)V;  // the vector's first column (padded rows: masking)
        odo_step<D, 1, false, IDX>(d, uo, off, oob);
      }
#pragma unroll
      for (int j = 0; j < K; ++j) {
        if (v + (IDX)j * dv < vend) {
          if (V > 1 && d.evpad) {  // padded odd rows: columns past the row are +0
            const IDX tau = d.t[0].tau;
#pragma unroll
            for (int e = 0; e < V; ++e) {
              if (colj[j] + (IDX)e < d.scols) {
                Mem<ESZ>::ld(addr<ESZ>(d.t[0].ptr, offj[j] + (IDX)e * tau), buf[j] + e * EW);
              } else {
#pragma unroll
                for (int q = 0; q < EW; ++q) buf[j][e * EW + q] = 0u;
              }
            }
          } else {
            load_vec<ESZ, V, IDX>(d.t[0], offj[j], lgL, buf[j]);
          }
        } else {
#pragma unroll
          for (int q = 0; q < NW; ++q) buf[j][q] = 0u;
        }
      }
#pragma unroll
      for (int j = 0; j < K; ++j) {
        if (v < vend) ev_accumulate<D, ESZ, V, IDX>(d, buf[j], a);
        digits_step_ev<D, IDX>(d, u, a);
        v += dv;
      }
    }
    ev_finish<D, IDX>(d, u, a, acc);
  }
  ev_reduce<NS, kBlock, IDX>(d, acc);
}

// ---- Blackwell bulk-copy pipeline primitives (cp.async.bulk + mbarrier; SASS: UBLKCP, SYNCS)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---- expected value, dense p with a short odd innermost extent n: rows through shared memory
// A vector is one row of n contiguous elements (plan.cpp plan_ev_rows); the digits are the outer
// axes.  Block b owns the contiguous tiles [b * wspan, (b+1) * wspan) of TR = kBlock * RPT rows;
// thread 0 keeps NST - 1 tiles in flight with 1-D bulk copies (cp.async.bulk, one mbarrier per
// stage completing on the transferred bytes) while all threads sum the current tile's rows from
// shared memory: thread t takes rows t, t + kBlock, ... -- one arithmetic progression of rows
// per thread across the block's tiles, so the digits advance by a fixed +kBlock rows step
// (digits_step_ev: the telescoped weights of ev_kernel, P:129's amortised carries).  Per row:
// mass s = sum_c x_c and column moment sum_c c x_c by suffix sums (T += x_c; m += T for c
// from n-1 down to 1), no per-element weight or odometer -- ~4 instructions per element
// against the flat kernel's ~10.  Bytes = p + d doubles.
// mass T and column moment m of one row of N elements by suffix sums, N a compile-time constant
template <int ESZ, int N>
__device__ __forceinline__ void ev_row_sums(const unsigned char* rp, double& T, double& m) {
#pragma unroll
  for (int c = N - 1; c >= 1; --c) {
    T += (double)Elem<ESZ>::get((const uint32_t*)(rp + c * ESZ));
    m += T;
  }
  T += (double)Elem<ESZ>::get((const uint32_t*)rp);
}

#ifndef TRIOT_EVROWS_MINB
#define TRIOT_EVROWS_MINB 2
#endif
#ifndef TRIOT_EVROWS_STAGE
#define TRIOT_EVROWS_STAGE 16384
#endif
constexpr int kEvRowsStages = 3;
template <int D, int ESZ, typename IDX>
__global__ void __launch_bounds__(kBlock, TRIOT_EVROWS_MINB)
    ev_rows_kernel(const __grid_constant__ Desc<IDX> d) {
  constexpr int NS = D + 2;  // D outer digits, the column moment, the mass
  constexpr int NST = kEvRowsStages;
  extern __shared__ __align__(128) unsigned char smem[];
  const uint32_t n = d.rowlen;
  const uint32_t RPT = d.rwin;       // rows per thread per tile
  const uint32_t stage = d.rmag;     // bytes per stage (multiple of 16)
  const IDX TR = (IDX)kBlock * (IDX)RPT;
  uint64_t* full = (uint64_t*)(smem + (size_t)NST * stage);
  const int tid = threadIdx.x;
  const IDX ntiles = (d.nvec + TR - 1) / TR;
  const IDX t0 = (IDX)blockIdx.x * d.wspan;
  IDX t1 = t0 + d.wspan;
  if (t1 > ntiles || t1 < t0) t1 = ntiles;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < NST; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  pdl_trigger();
  pdl_wait();
  __syncthreads();
  const char* pbase = (const char*)d.t[0].ptr;
  const uint64_t row_bytes = (uint64_t)n * ESZ;
  auto issue = [&](IDX tile, int s) {
    const IDX r0 = tile * TR;
    const IDX nr = (d.nvec - r0) < TR ? (d.nvec - r0) : TR;
    // round the last tile up to 16 bytes: the extra bytes lie in the same 16-byte granule as
    // p's last element (p is 16-byte aligned), are never summed, and cannot cross a page
    const uint32_t bytes = (uint32_t)(((uint64_t)nr * row_bytes + 15u) & ~15ull);
    mbar_expect_tx(&full[s], bytes);
    bulk_g2s(smem + (size_t)s * stage, pbase + (uint64_t)r0 * row_bytes, bytes, &full[s]);
  };
  if (tid == 0)
    for (int s = 0; s < NST - 1; ++s)
      if (t0 + (IDX)s < t1) issue(t0 + (IDX)s, s);
  const bool grp = d.rgroup != 0;  // a thread's rows of a tile: consecutive, or strided by the block
  IDX u[D];
  decode_digits<D, IDX>(d, t0 * TR + (grp ? (IDX)tid * (IDX)RPT : (IDX)tid), u);
  EvAcc<D> a;
  ev_acc_init<D, IDX>(a);
  for (IDX i = t0; i < t1; ++i) {
    const int s = (int)((i - t0) % NST);
    const uint32_t par = (uint32_t)(((i - t0) / NST) & 1);
    if (tid == 0 && i + (IDX)(NST - 1) < t1)  // its stage was released at the last barrier
      issue(i + (IDX)(NST - 1), (int)((i - t0 + NST - 1) % NST));
    mbar_wait(&full[s], par);
    const unsigned char* st = smem + (size_t)s * stage;
    for (uint32_t r = 0; r < RPT; ++r) {
      const uint32_t rit = grp ? (uint32_t)tid * RPT + r : r * kBlock + (uint32_t)tid;
      const IDX row = i * TR + (IDX)rit;
      if (row < d.nvec) {
        const unsigned char* rp = st + (size_t)rit * row_bytes;
        double T = 0.0, m = 0.0;
        // short rows fully unrolled (a run-time trip count costs more than their data: f32 rows
        // of 3 ran 79 instructions per row, ncu); longer ones the generic loop
        switch (n) {
          case 3: ev_row_sums<ESZ, 3>(rp, T, m); break;
          case 5: ev_row_sums<ESZ, 5>(rp, T, m); break;
          case 6: ev_row_sums<ESZ, 6>(rp, T, m); break;
          case 7: ev_row_sums<ESZ, 7>(rp, T, m); break;
          case 9: ev_row_sums<ESZ, 9>(rp, T, m); break;
          case 10: ev_row_sums<ESZ, 10>(rp, T, m); break;
          case 11: ev_row_sums<ESZ, 11>(rp, T, m); break;
          case 12: ev_row_sums<ESZ, 12>(rp, T, m); break;
          case 13: ev_row_sums<ESZ, 13>(rp, T, m); break;
          case 14: ev_row_sums<ESZ, 14>(rp, T, m); break;
          case 15: ev_row_sums<ESZ, 15>(rp, T, m); break;
          default:
#pragma unroll 4
            for (int c = (int)n - 1; c >= 1; --c) {
              T += (double)Elem<ESZ>::get((const uint32_t*)(rp + (size_t)c * ESZ));
              m += T;
            }
            T += (double)Elem<ESZ>::get((const uint32_t*)rp);
        }
        a.S += T;
        a.Wc += m;
      }
      if (grp && r + 1 < RPT) {
        // the next row of the group: Alg 3's +1 on the outer digits, each change
        // with its telescoped weight event -- one subtraction unless a digit wraps
#pragma unroll
        for (int k = D - 1; k >= 0; --k) {
          const IDX old = u[k];
          IDX nu = old + 1;
          const bool carry = k > 0 && nu >= d.ext[k];
          if (carry) nu = 0;
          u[k] = nu;
          a.ev[k] = carry ? fma((double)old, a.S, a.ev[k]) : a.ev[k] - a.S;
          if (!carry) break;
        }
      } else {
        digits_step_ev<D, IDX>(d, u, a);
      }
    }
    __syncthreads();  // every thread is done with stage s before thread 0 refills it
  }
  double acc[NS];
#pragma unroll
  for (int k = 0; k < D; ++k) acc[k] = fma((double)u[k], a.S, a.ev[k]);
  acc[D] = a.Wc;
  acc[D + 1] = a.S;
  ev_reduce<NS, kBlock, IDX>(d, acc);
}

// ---- expected value of a view window with long rows (n in 32..256): TMA tensor tiles
// A window of a base tensor has contiguous rows at the base's strides; a TMA tensor map over the
// base (rank m = the window's axes of extent > 1, at most 5) moves boxes of R rows x nbox
// columns (nbox = n rounded up to 16 bytes; columns past the base are zero-filled by the TMA,
// columns past the window masked) into a 3-stage shared-memory ring, thread 0 issuing
// `cp.async.bulk.tensor` for tile i + 2 while the block consumes tile i.  Thread t owns column
// t of every row: per element one shared load and one fp64 add into its running column mass S;
// the outer digits' weights are telescoped over its row sequence (+1 row inside a tile, a jump
// between tiles: one FMA per change, P:129's argument) and the column weight t multiplies S
// once at the end -- no per-element weight, odometer or offset arithmetic.
struct EvTmaGeo {
  uint64_t ext[4];    // window extents of the outer axes (digits 0..D-1; digit D-1 = the row axis)
  int32_t coord0[5];  // base coordinate of the window start per TMA dim (dim 0 = innermost)
  uint32_t m;         // TMA rank (D + 1)
  uint32_t n, nbox, R, stage;
  uint32_t cshift;    // columns the box starts before the window (16-byte aligned box start)
  uint64_t tpa;       // tiles along the row axis: ceil(ext[D-1] / R)
  uint64_t ntiles, per;
};

__device__ __forceinline__ void tma_load_tile(void* dst, const void* map, int m, const int32_t* c,
                                              uint64_t* bar) {
  const uint32_t sd = smem_u32(dst), sb = smem_u32(bar);
  const uint64_t mp = (uint64_t)map;
  switch (m) {
    case 2:
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3}], [%4];" ::"r"(sd), "l"(mp), "r"(c[0]), "r"(c[1]), "r"(sb)
          : "memory");
      break;
    case 3:
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(sd), "l"(mp), "r"(c[0]), "r"(c[1]), "r"(c[2]),
          "r"(sb)
          : "memory");
      break;
    case 4:
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(sd), "l"(mp), "r"(c[0]), "r"(c[1]),
          "r"(c[2]), "r"(c[3]), "r"(sb)
          : "memory");
      break;
    default:
      asm volatile(
          "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(sd), "l"(mp), "r"(c[0]), "r"(c[1]),
          "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(sb)
          : "memory");
      break;
  }
}

template <int D, int ESZ>
__global__ void __launch_bounds__(kBlock, 4)
    ev_view_tma_kernel(const __grid_constant__ Desc<uint32_t> d,
                       const __grid_constant__ CUtensorMap map, const __grid_constant__ EvTmaGeo G) {
  constexpr int NS = D + 2;  // the outer digits, the column moment, the mass
  constexpr int NST = kEvRowsStages;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = (uint64_t*)(smem + (size_t)NST * G.stage);
  const int tid = threadIdx.x;
  const uint64_t t0 = (uint64_t)blockIdx.x * G.per;
  uint64_t t1 = t0 + G.per;
  if (t1 > G.ntiles) t1 = G.ntiles;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < NST; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&map) : "memory");
  }
  pdl_trigger();
  pdl_wait();
  __syncthreads();
  // tile position as an odometer: a = tile index along the row axis, pre[] = the digits of the
  // axes above it (32-bit: ntiles < 2^32 is checked on the host); one division per thread at
  // the start, then +1 tile steps -- 64-bit divisions per tile cost more than the tile's work
  struct Pos {
    uint32_t a;
    uint32_t pre[D > 1 ? D - 1 : 1];
  };
  auto pos_of = [&](uint64_t tile) {
    Pos q;
    uint32_t t = (uint32_t)tile;
    q.a = t % (uint32_t)G.tpa;
    t /= (uint32_t)G.tpa;
#pragma unroll
    for (int k = D - 2; k >= 0; --k) {
      q.pre[k] = t % (uint32_t)G.ext[k];
      t /= (uint32_t)G.ext[k];
    }
    return q;
  };
  auto advance = [&](Pos& q) {
    if (++q.a == (uint32_t)G.tpa) {
      q.a = 0;
#pragma unroll
      for (int k = D - 2; k >= 0; --k) {
        if (++q.pre[k] < (uint32_t)G.ext[k]) break;
        q.pre[k] = 0;
      }
    }
  };
  auto issue = [&](const Pos& q, int s) {
    int32_t c[5];
    c[0] = G.coord0[0];
    c[1] = G.coord0[1] + (int32_t)(q.a * G.R);
#pragma unroll
    for (int j = 2; j <= D; ++j) c[j] = G.coord0[j] + (int32_t)q.pre[D - j];
    mbar_expect_tx(&full[s], G.nbox * G.R * ESZ);
    tma_load_tile(smem + (size_t)s * G.stage, &map, (int)G.m, c, &full[s]);
  };
  Pos ip;  // thread 0: the next tile to issue
  if (tid == 0 && t0 < t1) {
    ip = pos_of(t0);
    for (int s = 0; s < NST - 1; ++s)
      if (t0 + (uint64_t)s < t1) {
        issue(ip, s);
        advance(ip);
      }
  }
  const bool active = (uint32_t)tid < G.n;
  Pos cp = pos_of(t0 < t1 ? t0 : 0);  // the tile being consumed
  uint32_t u[D];
#pragma unroll
  for (int k = 0; k < D - 1; ++k) u[k] = cp.pre[k];
  u[D - 1] = cp.a * G.R;
  double S = 0.0, ev[D];
#pragma unroll
  for (int k = 0; k < D; ++k) ev[k] = 0.0;
  for (uint64_t i = t0; i < t1; ++i) {
    const int s = (int)((i - t0) % NST);
    const uint32_t par = (uint32_t)(((i - t0) / NST) & 1);
    if (tid == 0 && i + (uint64_t)(NST - 1) < t1) {
      issue(ip, (int)((i - t0 + NST - 1) % NST));
      advance(ip);
    }
    // jump to the tile's first row: one event per changed digit
#pragma unroll
    for (int k = 0; k < D - 1; ++k)
      if (cp.pre[k] != u[k]) {
        ev[k] = fma(-((double)cp.pre[k] - (double)u[k]), S, ev[k]);
        u[k] = cp.pre[k];
      }
    {
      const uint32_t r0 = cp.a * G.R;
      if (r0 != u[D - 1]) {
        ev[D - 1] = fma(-((double)r0 - (double)u[D - 1]), S, ev[D - 1]);
        u[D - 1] = r0;
      }
    }
    const uint32_t left = (uint32_t)G.ext[D - 1] - cp.a * G.R;
    const uint32_t rows = left < G.R ? left : G.R;
    mbar_wait(&full[s], par);
    const unsigned char* st = smem + (size_t)s * G.stage + (size_t)(tid + G.cshift) * ESZ;
    const uint32_t pitch = G.nbox * ESZ;
    if (active) {
      S += (double)Elem<ESZ>::get((const uint32_t*)st);
      for (uint32_t r = 1; r < rows; ++r) {  // next row: the row digit + 1
        ev[D - 1] -= S;
        S += (double)Elem<ESZ>::get((const uint32_t*)(st + r * pitch));
      }
    }
    u[D - 1] += rows - 1;
    advance(cp);
    __syncthreads();  // stage s consumed before thread 0 refills it
  }
  double acc[NS];
#pragma unroll
  for (int k = 0; k < D; ++k) acc[k] = fma((double)u[k], S, ev[k]);
  acc[D] = (double)tid * S;  // column weight t times the column's mass
  acc[D + 1] = S;
  ev_reduce<NS, kBlock, uint32_t>(d, acc);
}

// ------------------------------------------------------------------ NEXT-2: inner product
// Benchmark 2 / Alg 8 dot_product: sum_t a[t] * b[t] over the iteration
// shape, each operand indexed by its own shape.  fp64 accumulation (one fused multiply-add per
// element), the EV's deterministic block/last-block reduction with one slot.
template <int D, int ESZ, int V, typename IDX, int K>
__global__ void __launch_bounds__(kBlock) dot_kernel(const __grid_constant__ Desc<IDX> d) {
  constexpr int EW = ESZ / 4;
  constexpr int NW = V * EW;
  const int lane = threadIdx.x & 31;
  const IDX warp = (IDX)blockIdx.x * (kBlock / 32) + (IDX)(threadIdx.x >> 5);
  const IDX base0 = warp * d.wmul;
  double acc[1] = {0.0};
  pdl_trigger();
  TRIOT_TRACE(0);
  if (base0 < d.nvec) {
    const IDX vend = warp_end(d, base0);
    IDX u[D], off[2];
    uint32_t oob;
    IDX v = base0 + (IDX)lane;
    odo_start<D, 2, false, IDX>(d, v, u, off, oob);
    const uint32_t lgL = d.lgL;
    pdl_wait();
    for (IDX b = base0; b < vend; b += K * d.dv) {
      uint32_t ba[K][NW], bb[K][NW];
      bool valid[K];
#pragma unroll
      for (int j = 0; j < K; ++j) {
        valid[j] = v < vend;
        v += d.dv;
        if (valid[j]) {
          load_vec<ESZ, V, IDX>(d.t[0], off[0], lgL, ba[j]);
          load_vec<ESZ, V, IDX>(d.t[1], off[1], lgL, bb[j]);
        }
        odo_step<D, 2, false, IDX>(d, u, off, oob);
      }
#pragma unroll
      for (int j = 0; j < K; ++j) {
        if (!valid[j]) continue;
#pragma unroll
        for (int e = 0; e < V; ++e)
          acc[0] = fma((double)Elem<ESZ>::get(ba[j] + e * EW),
                       (double)Elem<ESZ>::get(bb[j] + e * EW), acc[0]);
      }
    }
  } else {
    pdl_wait();
  }
  TRIOT_TRACE(2);
  ev_reduce<1, kBlock, IDX>(d, acc);
  TRIOT_TRACE(4);
}

// ------------------------------------------------------------------ NEXT-3: fused update
// Benchmark 3: x[t] <- x[t] + y[t] * x[t] - z[t] for every t of x's shape, in place on x
// (the aliasing-safe apply_tensors idiom).  C evaluation order with one rounding per
// operation: (x + (y * x)) - z.  Tensor 0 = x, 1 = y, 2 = z.
template <int D, int ESZ, int V, typename IDX, int K>
__global__ void __launch_bounds__(kBlock) update_kernel(const __grid_constant__ Desc<IDX> d) {
  constexpr int EW = ESZ / 4;
  constexpr int NW = V * EW;
  using T = typename Elem<ESZ>::T;
  const int lane = threadIdx.x & 31;
  const IDX warp = (IDX)blockIdx.x * (kBlock / 32) + (IDX)(threadIdx.x >> 5);
  const IDX base0 = warp * d.wmul;
  pdl_trigger();
  if (base0 >= d.nvec) return;
  const IDX vend = warp_end(d, base0);
  IDX u[D], off[3];
  uint32_t oob;
  IDX v = base0 + (IDX)lane;
  odo_start<D, 3, false, IDX>(d, v, u, off, oob);
  const uint32_t lgL = d.lgL;
  pdl_wait();
  for (IDX b = base0; b < vend; b += K * d.dv) {
    uint32_t bx[K][NW], by[K][NW], bz[K][NW];
    IDX xoff[K];
    bool valid[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      valid[j] = v < vend;
      v += d.dv;
      xoff[j] = off[0];
      if (valid[j]) {
        load_vec<ESZ, V, IDX, false>(d.t[0], off[0], lgL, bx[j]);
        load_vec<ESZ, V, IDX, false>(d.t[1], off[1], lgL, by[j]);
        load_vec<ESZ, V, IDX, false>(d.t[2], off[2], lgL, bz[j]);
      }
      odo_step<D, 3, false, IDX>(d, u, off, oob);
    }
#pragma unroll
    for (int j = 0; j < K; ++j) {
      if (!valid[j]) continue;
      uint32_t r[NW];
#pragma unroll
      for (int e = 0; e < V; ++e) {
        const T x = Elem<ESZ>::get(bx[j] + e * EW);
        const T yx = bop<2>(Elem<ESZ>::get(by[j] + e * EW), x);
        Elem<ESZ>::put(r + e * EW, bop<1>(bop<0>(x, yx), Elem<ESZ>::get(bz[j] + e * EW)));
      }
      store_vec<ESZ, V, IDX>(d.t[0], xoff[j], lgL, r);
    }
  }
}

// EV on flat vectors (odd innermost extents): p is the counter itself, so vector v is elements
// [v*V, v*V + V) of p; the element digits are the weights, walked with the +1 odometer and its
// deferred-weight events.
// VB = 64 (rows longer than a unit, so at most one wrap per unit): two 32-byte loads per lane
// and unit; the unit's mass and its sum of prefix sums come from one pass of adds and
// immediate-weight FMAs (no prefix array), the prefix at the wrap from a second pass
// of block masses plus at most three elements, taken only by the warps in which a lane wraps;
// the digit bookkeeping is paid once per 64 bytes (rows of 33, 268 MB, ncu cold: f32 65.6 ->
// 51.5-53.3 us = 5.0-5.2 TB/s, 154 -> 103 warp instructions per 32 bytes; f64 54.2 -> 46.9 us
// = 5.7 TB/s, 129 -> 78; profiles/r02_evodd_flat*).
template <int D, int ESZ, typename IDX, int K, int VB = 32>
__global__ void __launch_bounds__(kBlock) ev_flat_kernel(const __grid_constant__ Desc<IDX> d) {
  constexpr int V = VB / ESZ;
  constexpr int EW = ESZ / 4;
  constexpr int NW = V * EW;
  constexpr int NS = D + 2;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const IDX warp = (IDX)blockIdx.x * (kBlock / 32) + (IDX)wib;
  const IDX base0 = warp * d.wmul;
  double acc[NS];
#pragma unroll
  for (int k = 0; k < NS; ++k) acc[k] = 0.0;
  pdl_trigger();
  pdl_wait();
  if (base0 < d.nvec) {
    const IDX vend = warp_end(d, base0);
    const IDX dv = d.dv;
    IDX v = base0 + (IDX)lane;
    IDX u[D];
    ev_decode<D, IDX>(d, v * (IDX)V, u);
    EvAcc<D> a;
    ev_acc_init<D, IDX>(a);
    const bool pvec = d.t[0].vec != 0;
    const double nd = (double)d.ext[D - 1];
    const uint32_t wmax = D > 1 ? (uint32_t)((IDX)V / d.ext[D - 1]) + 1u : 0u;  // wraps <= this
    for (IDX b = base0; b < vend; b += (IDX)K * dv) {
      uint32_t buf[K][NW];
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const IDX vj = v + (IDX)j * dv;
        const IDX f0 = vj * (IDX)V;
        if (vj < vend && pvec && f0 + (IDX)V <= d.nelem) {
          Mem<32>::ld(addr<ESZ>(d.t[0].ptr, f0), buf[j]);
          if constexpr (VB == 64)
            Mem<32>::ld(addr<ESZ>(d.t[0].ptr, f0 + (IDX)(V / 2)), buf[j] + NW / 2);
        } else {
#pragma unroll
          for (int e = 0; e < V; ++e) {
            if (vj < vend && f0 + (IDX)e < d.nelem) {
              Mem<ESZ>::ld(addr<ESZ>(d.t[0].ptr, f0 + (IDX)e), buf[j] + e * EW);
            } else {
#pragma unroll
              for (int q = 0; q < EW; ++q) buf[j][e * EW + q] = 0u;
            }
          }
        }
      }
#pragma unroll
      for (int j = 0; j < K; ++j) {
        // V elements, each followed by Alg 3's +1 with its weight events in closed
        // form: every +1 of the innermost digit contributes -1 x (running mass), i.e.
        // -(V S + sum of the V prefix sums) in total; a wrap (column n-1 -> 0) instead changes
        // it by -(n-1), a correction of +n x (mass at the wrap), and carries into the outer
        // digits with their own events.  Past the end the elements are +0.0.
        const IDX col = u[D - 1];
        IDX ew = D > 1 ? d.ext[D - 1] - col : (IDX)(V + 1);
        double pre, sumpre;
        double pfx[VB == 64 ? 1 : V + 1];  // pfx[e] = sum of the vector's first e elements
        constexpr int NB = VB == 64 ? V / 4 : 1;  // blocks of four elements (VB = 64)
        double sb[NB];
        if constexpr (VB == 64) {
          // block masses, the unit's mass and the sum of the V prefix sums (= sum_e (V - e) x_e)
          // in one pass
          double q0 = 0.0, q1 = 0.0;
#pragma unroll
          for (int b = 0; b < NB; ++b) {
            const double x0 = (double)Elem<ESZ>::get(buf[j] + (4 * b) * EW);
            const double x1 = (double)Elem<ESZ>::get(buf[j] + (4 * b + 1) * EW);
            const double x2 = (double)Elem<ESZ>::get(buf[j] + (4 * b + 2) * EW);
            const double x3 = (double)Elem<ESZ>::get(buf[j] + (4 * b + 3) * EW);
            sb[b] = (x0 + x1) + (x2 + x3);
            q0 = fma((double)(V - 4 * b), x0, q0);
            q1 = fma((double)(V - 4 * b - 1), x1, q1);
            q0 = fma((double)(V - 4 * b - 2), x2, q0);
            q1 = fma((double)(V - 4 * b - 3), x3, q1);
          }
          pre = sb[0];
#pragma unroll
          for (int b = 1; b < NB; ++b) pre += sb[b];
          sumpre = q0 + q1;
        } else {
          pfx[0] = 0.0;
          sumpre = 0.0;
#pragma unroll
          for (int e = 0; e < V; ++e) {
            pfx[e + 1] = pfx[e] + (double)Elem<ESZ>::get(buf[j] + e * EW);
            sumpre += pfx[e + 1];
          }
          pre = pfx[V];
        }
        // wraps (column n-1 -> 0) follow elements ew - 1 with ew = n - col, ew + n, ... <= V;
        // the loop trip count is uniform (V / n + 1), so the warp stays converged
        for (uint32_t w = 0; w < wmax; ++w, ew += d.ext[D - 1]) {
          if (ew > (IDX)V) continue;
          double pw = 0.0;  // the sum of the first ew elements (ew is per lane)
          if constexpr (VB == 64) {
            // whole blocks before the wrap, then up to three elements of the block it falls in
            // (its raw words picked by a select chain over the blocks: no dynamic indexing)
            const uint32_t bw = (uint32_t)ew >> 2, r = (uint32_t)ew & 3u;
#pragma unroll
            for (int b = 0; b < NB; ++b) pw += ((uint32_t)b < bw) ? sb[b] : 0.0;
#pragma unroll
            for (int i = 0; i < 3; ++i) {
              uint32_t raw[EW];
#pragma unroll
              for (int q = 0; q < EW; ++q) raw[q] = buf[j][(4 * (NB - 1) + i) * EW + q];
#pragma unroll
              for (int b = NB - 2; b >= 0; --b)
#pragma unroll
                for (int q = 0; q < EW; ++q)
                  raw[q] = ((uint32_t)b == bw) ? buf[j][(4 * b + i) * EW + q] : raw[q];
              pw += ((uint32_t)i < r) ? (double)Elem<ESZ>::get(raw) : 0.0;
            }
          } else {
#pragma unroll
            for (int e = 1; e <= V; ++e) pw = ((IDX)e == ew) ? pfx[e] : pw;
          }
          const double sc = a.S + pw;  // the running mass at this wrap
          a.ev[D - 1] = fma(nd, sc, a.ev[D - 1]);
#pragma unroll
          for (int k = D - 2; k >= 0; --k) {
            const IDX old = u[k];
            IDX nu = old + 1;
            const bool carry = k > 0 && nu >= d.ext[k];
            if (carry) nu = 0;
            u[k] = nu;
            a.ev[k] = fma(-(double)((int64_t)nu - (int64_t)old), sc, a.ev[k]);
            if (!carry) break;
          }
        }
        {
          // col + V - n * (number of wraps)
          IDX c2 = col + (IDX)V;
          while (D > 1 && c2 >= d.ext[D - 1]) c2 -= d.ext[D - 1];
          u[D - 1] = c2;
        }
        a.ev[D - 1] -= fma((double)V, a.S, sumpre);
        a.S += pre;
        digits_step_ev<D, IDX>(d, u, a);
        v += dv;
      }
    }
#pragma unroll
    for (int k = 0; k < D; ++k) acc[k] = fma((double)u[k], a.S, a.ev[k]);
    acc[D] = 0.0;
    acc[D + 1] = a.S;
  }
  ev_reduce<NS, kBlock, IDX>(d, acc);
}

// ------------------------------------------------------------------ NEXT-4: naive convolution
// Alg 15: result[t_l + t_r] += lhs[t_l] * rhs[t_r].  Output-stationary: each output
// tuple u gathers every (t_l, u - t_l) pair -- the valid t_l form a box
// [max(0, u_k - R_k + 1), min(L_k - 1, u_k)] per axis -- in lexicographic order of t_l, adding
// each rounded product in exactly the order Alg 15's outer enumerate visits t_l, so the result
// is bit-identical to the sequential algorithm (and needs no atomics).  Descriptor use: ext / fdm / fds = result shape; t[0].sig = lhs strides,
// t[1].sig = rhs strides, t[2].sig = result strides; bnd[k] = lhs extents, dlt[k] = rhs extents.
// Operand access for the convolution: shared memory through 32-bit shared-window addresses
// (ld.shared; generic pointers into shared memory made the compiler rebuild the window address
// every iteration) or global memory through the read-only path.
template <typename T, bool SMEM>
struct ConvSrc {
  const T* g;
  uint32_t s;  // shared-window byte address
  __device__ __forceinline__ T at(uint32_t i) const {
    if (SMEM) {
      T v;
      if (sizeof(T) == 8)
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(*(double*)&v) : "r"(s + i * 8u));
      else
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(*(float*)&v) : "r"(s + i * 4u));
      return v;
    }
    return __ldg(g + i);
  }
};

// A group of G consecutive lanes per output tuple u.  The output's terms are its box of valid
// t_l in lexicographic order; lane j of the group takes terms j, j+G, ... (its box tuple
// advances by +G in the box's mixed radix: the Alg 3 odometer with per-output extents) and forms
// the rounded product; each round the group folds its G products in term order (width-G
// shuffles) into the one dependent add chain -- exactly Alg 15's sequence of additions.
// Invalid lanes contribute +0.0, which never changes the sum (it starts at +0.0, so it can
// never be -0.0).  G = 8: the shuffle/add issue per term stays low (4 outputs share a warp) and
// each round's 8-add chain hides the pipelined loads, products and shuffles of later rounds.
template <int D, int G, typename T, typename Src>
__device__ __forceinline__ T conv_group(const Desc<uint32_t>& d, const Src& L, const Src& R,
                                        const uint32_t (&u)[D], int j, bool active) {
  uint32_t lo[D], ext[D], dig[D], dl[D];
  uint64_t M = 1;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const uint32_t Lk = d.bnd[k], Rk = d.dlt[k];
    lo[k] = u[k] + 1 > Rk ? u[k] + 1 - Rk : 0;
    const uint32_t hik = u[k] < Lk - 1 ? u[k] : Lk - 1;
    ext[k] = hik - lo[k] + 1;
    M *= ext[k];
  }
  if (!active) M = 0;
  uint32_t jj = (uint32_t)j, st = (uint32_t)G;
#pragma unroll
  for (int k = D - 1; k >= 0; --k) {
    dig[k] = jj % ext[k];
    jj /= ext[k];
    dl[k] = st % ext[k];
    st /= ext[k];
  }
  uint32_t offL = 0, offR = 0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    offL += (lo[k] + dig[k]) * d.t[0].sig[k];
    offR += (u[k] - lo[k] - dig[k]) * d.t[1].sig[k];
  }
  auto advance = [&]() {  // the lane's term += G (mixed-radix add; past the end never used)
    uint32_t c = 0;
#pragma unroll
    for (int k = D - 1; k >= 0; --k) {
      uint32_t nd = dig[k] + dl[k] + c;
      c = nd >= ext[k] ? 1u : 0u;
      if (c) nd -= ext[k];
      const int32_t delta = (int32_t)nd - (int32_t)dig[k];
      offL += (uint32_t)(delta * (int32_t)d.t[0].sig[k]);
      offR -= (uint32_t)(delta * (int32_t)d.t[1].sig[k]);
      dig[k] = nd;
    }
  };
  // Software pipeline over rounds r (G terms each): loads run two rounds ahead, the product and
  // its shuffles one round ahead, so in program order the dependent add chain of round r is
  // followed by work that does not wait on it.
  // branch-free loads: a lane past its box loads element 0 and its product is replaced by +0.0
  // The group's G products of a round reach every lane of the group through a per-warp
  // double-buffered shared-memory slot (one store per lane, G/2 16-byte loads) instead of G
  // shuffles; the __syncwarp after each round's stores orders them before the next round's loads
  // and after the previous round's loads of the same buffer.
  __shared__ __align__(16) T xbuf[TRIOT_CONV_BLOCK / 32][2][32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, g0 = lane - j;
  uint64_t term = (uint64_t)j;  // this lane's term index for the loads being issued
  bool va = term < M;
  T la = L.at(va ? offL : 0u), ra = R.at(va ? offR : 0u);   // round 0
  advance();
  term += G;
  xbuf[w][0][lane] = va ? bop<2>(la, ra) : T(0);
  __syncwarp();
  va = term < M;
  la = L.at(va ? offL : 0u);
  ra = R.at(va ? offR : 0u);   // round 1
  advance();
  term += G;
  // products of round 0 -> registers (the loop loads round r+1's right after its __syncwarp, so
  // the shared-memory latency overlaps the next round's operand loads)
  T q[G];
  auto fetch = [&](int buf) {
    if constexpr (sizeof(T) == 8) {
      const double2* x2 = reinterpret_cast<const double2*>(&xbuf[w][buf][g0]);
#pragma unroll
      for (int i = 0; i < G / 2; ++i) {
        const double2 v = x2[i];
        q[2 * i] = v.x;
        q[2 * i + 1] = v.y;
      }
    } else {
      const float4* x4 = reinterpret_cast<const float4*>(&xbuf[w][buf][g0]);
#pragma unroll
      for (int i = 0; i < G / 4; ++i) {
        const float4 v = x4[i];
        q[4 * i] = v.x;
        q[4 * i + 1] = v.y;
        q[4 * i + 2] = v.z;
        q[4 * i + 3] = v.w;
      }
    }
  };
  fetch(0);
  T acc = T(0);
  int cur = 0;
  for (uint64_t base = 0; __any_sync(0xffffffffu, base < M); base += G) {
    // a. loads of round r+2
    const bool vb = term < M;
    const T lb = L.at(vb ? offL : 0u), rb = R.at(vb ? offR : 0u);
    // b. the ordered add chain of round r (+0.0 for terms past the box)
#pragma unroll
    for (int i = 0; i < G; ++i) acc = bop<0>(acc, q[i]);
    // c. product of round r+1 into the other buffer, then its G products into registers
    xbuf[w][cur ^ 1][lane] = va ? bop<2>(la, ra) : T(0);
    __syncwarp();
    cur ^= 1;
    fetch(cur);
    la = lb;
    ra = rb;
    va = vb;
    advance();
    term += G;
  }
  return acc;
}

// Both operands into shared memory: two bulk copies of their 16-B-aligned prefixes (mbarrier
// complete_tx) plus element copies of the tails.  Calls griddepcontrol.wait before reading.
template <typename T, int BLOCK>
__device__ __forceinline__ void conv_stage(const Desc<uint32_t>& d, const T* lhs, const T* rhs,
                                           T* sl, T* sr) {
  constexpr int ESZ = (int)sizeof(T);
  __shared__ __align__(8) uint64_t bar;
  const uint32_t nl = (uint32_t)d.t[0].rho, nr = (uint32_t)d.t[1].rho;
  const bool al = ((uintptr_t)lhs & 15u) == 0, ar = ((uintptr_t)rhs & 15u) == 0;
  const uint32_t bl = al ? (nl * ESZ) & ~15u : 0u, br = ar ? (nr * ESZ) & ~15u : 0u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();
  if (threadIdx.x == 0 && bl + br) {
    mbar_expect_tx(&bar, bl + br);
    if (bl) bulk_g2s(sl, lhs, bl, &bar);
    if (br) bulk_g2s(sr, rhs, br, &bar);
  }
  for (uint32_t i = bl / ESZ + threadIdx.x; i < nl; i += BLOCK) sl[i] = __ldg(lhs + i);
  for (uint32_t i = br / ESZ + threadIdx.x; i < nr; i += BLOCK) sr[i] = __ldg(rhs + i);
  if (bl + br) mbar_wait(&bar, 0);
  __syncthreads();
}

// Lane per output (the default).  Tensor 0 is the operand whose index space is iterated (A),
// tensor 1 the other (B); bnd / dlt = their extents.  The 32 outputs of a warp iterate the union
// of their boxes of valid A-tuples (warp-uniform odometer: A's offsets are uniform, so its loads
// are shared-memory broadcasts) with a per-lane validity mask; an invalid term adds +0.0, which
// leaves the sum unchanged (it starts at +0.0 and so is never -0.0).  Forward lexicographic order
// when A = lhs; when A = rhs (the host picks the smaller operand as A) the order is reversed,
// which is lexicographic in t_l = u - t_r.  Either way each output adds its rounded products in
// exactly Alg 15's order: bit-identical to the sequential algorithm, one add chain per lane.
constexpr int kConvLaneBlock = 64;
template <int D, int ESZ, bool SMEM, bool REV>
__global__ void __launch_bounds__(kConvLaneBlock) conv_lane_kernel(
    const __grid_constant__ Desc<uint32_t> d) {
  using T = typename Elem<ESZ>::T;
  pdl_trigger();
  const T* ga = (const T*)d.t[0].ptr;
  const T* gb = (const T*)d.t[1].ptr;
  extern __shared__ __align__(128) unsigned char conv_smem[];
  T* sa = (T*)conv_smem;
  T* sb = sa + d.t[0].numel_pad;
  if (SMEM) conv_stage<T, kConvLaneBlock>(d, ga, gb, sa, sb);
  else pdl_wait();
  const ConvSrc<T, SMEM> A{ga, SMEM ? smem_u32(sa) : 0u}, B{gb, SMEM ? smem_u32(sb) : 0u};
  const uint32_t uf = blockIdx.x * kConvLaneBlock + threadIdx.x;
  const bool active = uf < d.nvec;
  uint32_t u[D], lo[D], hi[D];
  {
    uint32_t r = active ? uf : 0u;
#pragma unroll
    for (int k = D - 1; k >= 1; --k) {
      const uint32_t q = divq<uint32_t>(r, d.ext[k], d.fdm[k], d.fds[k]);
      u[k] = r - q * d.ext[k];
      r = q;
    }
    u[0] = r;
  }
  uint32_t baseB = 0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const uint32_t Ak = d.bnd[k], Bk = d.dlt[k];
    lo[k] = active ? (u[k] + 1 > Bk ? u[k] + 1 - Bk : 0u) : 0xffffffffu;
    hi[k] = active ? (u[k] < Ak - 1 ? u[k] : Ak - 1) : 0u;
    baseB += u[k] * d.t[1].sig[k];
  }
  uint32_t ulo[D], uhi[D], t[D];
#pragma unroll
  for (int k = 0; k < D; ++k) {
    ulo[k] = __reduce_min_sync(0xffffffffu, lo[k]);
    uhi[k] = __reduce_max_sync(0xffffffffu, hi[k]);
    t[k] = REV ? uhi[k] : ulo[k];
  }
  if (ulo[0] > uhi[0]) return;  // no active output in this warp
  const uint32_t sA = d.t[0].sig[D - 1], sB = d.t[1].sig[D - 1];
  const uint32_t n = uhi[D - 1] - ulo[D - 1] + 1;  // terms per row of the union box
  const uint32_t ilo = lo[D - 1], ihi = hi[D - 1];
  // The union box is walked in chunks of RB terms along its rows (a chunk never crosses a row;
  // a row's last chunk is padded with +0.0 terms).  Software pipeline: the next chunk's loads are
  // issued before the current chunk's products join the add chain, so the chain -- one dependent
  // add per term, Alg 15's order -- is the critical path.
  constexpr int RB = 8;
  struct Chunk {
    uint32_t offA, idxB, ti, rem;  // A offset / B index of the first term, its inner digit,
    bool vo, live;                 // terms left in the row; outer digits in this lane's box
  };
  auto row_start = [&](Chunk& c) {
    uint32_t hB = 0;
    c.offA = 0;
    c.vo = true;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      c.offA += t[k] * d.t[0].sig[k];
      hB += t[k] * d.t[1].sig[k];
      if (k < D - 1) c.vo = c.vo && t[k] >= lo[k] && t[k] <= hi[k];
    }
    c.idxB = baseB - hB;
    c.ti = t[D - 1];
    c.rem = n;
    c.live = true;
  };
  auto advance = [&](Chunk& c) {
    if (c.rem > (uint32_t)RB) {
      c.rem -= RB;
      if (REV) {
        c.ti -= RB;
        c.offA -= RB * sA;
        c.idxB += RB * sB;
      } else {
        c.ti += RB;
        c.offA += RB * sA;
        c.idxB -= RB * sB;
      }
      return;
    }
    // next row of the union box: Alg 3's carry on digits 0..D-2 (a borrow when reversed)
    bool carry = true;
#pragma unroll
    for (int k = D - 2; k >= 0; --k) {
      if (carry) {
        if (REV ? t[k] > ulo[k] : t[k] < uhi[k]) {
          t[k] = REV ? t[k] - 1 : t[k] + 1;
          carry = false;
        } else {
          t[k] = REV ? uhi[k] : ulo[k];
        }
      }
    }
    if (carry) {
      c.live = false;
      return;
    }
    row_start(c);
  };
  auto issue = [&](const Chunk& c, T (&xa)[RB], T (&xb)[RB], bool (&xv)[RB]) {
#pragma unroll
    for (int q = 0; q < RB; ++q) {
      const bool inrow = c.live && (uint32_t)q < c.rem;
      const uint32_t tq = REV ? c.ti - q : c.ti + q;
      xv[q] = inrow && c.vo && tq >= ilo && tq <= ihi;
      xa[q] = A.at(inrow ? (REV ? c.offA - q * sA : c.offA + q * sA) : 0u);
      xb[q] = B.at(xv[q] ? (REV ? c.idxB + q * sB : c.idxB - q * sB) : 0u);
    }
  };
  Chunk c;
  row_start(c);
  T xa[RB], xb[RB];
  bool xv[RB];
  issue(c, xa, xb, xv);
  T acc = T(0);
  while (c.live) {
    Chunk nc = c;
    advance(nc);
    T ya[RB], yb[RB];
    bool yv[RB];
    issue(nc, ya, yb, yv);
#pragma unroll
    for (int q = 0; q < RB; ++q) acc = bop<0>(acc, xv[q] ? bop<2>(xa[q], xb[q]) : T(0));
    c = nc;
#pragma unroll
    for (int q = 0; q < RB; ++q) {
      xa[q] = ya[q];
      xb[q] = yb[q];
      xv[q] = yv[q];
    }
  }
  if (active) ((T*)d.out)[uf] = acc;
}

// Group variant (policy mode 1): G lanes per output.  SMEM: lhs and rhs are first copied into
// shared memory by two bulk copies (they are re-read by every output of the block; the paper's
// (2^8, 2^3) operands are 16 KB each).
template <int D, int ESZ, bool SMEM>
__global__ void __launch_bounds__(TRIOT_CONV_BLOCK) conv_kernel(
    const __grid_constant__ Desc<uint32_t> d) {
  using T = typename Elem<ESZ>::T;
  constexpr int G = TRIOT_CONV_GROUP;
  const int j = threadIdx.x % G;
  const uint32_t u_flat = blockIdx.x * (TRIOT_CONV_BLOCK / G) + threadIdx.x / G;
  pdl_trigger();
  const T* lhs = (const T*)d.t[0].ptr;
  const T* rhs = (const T*)d.t[1].ptr;
  extern __shared__ __align__(128) unsigned char conv_smem[];
  T* sl = (T*)conv_smem;
  T* sr = sl + d.t[0].numel_pad;
  if (SMEM) conv_stage<T, TRIOT_CONV_BLOCK>(d, lhs, rhs, sl, sr);
  // every lane stays to the end (the group shuffles need the full warp); past-the-end groups
  // compute nothing
  const bool active = u_flat < d.nvec;
  uint32_t u[D];
  {
    uint32_t r = active ? u_flat : 0u;
#pragma unroll
    for (int k = D - 1; k >= 1; --k) {
      const uint32_t q = divq<uint32_t>(r, d.ext[k], d.fdm[k], d.fds[k]);
      u[k] = r - q * d.ext[k];
      r = q;
    }
    u[0] = r;
  }
  T acc;
  if (SMEM) {
    const ConvSrc<T, true> Ls{nullptr, smem_u32(sl)}, Rs{nullptr, smem_u32(sr)};
    acc = conv_group<D, G, T>(d, Ls, Rs, u, j, active);
  } else {
    pdl_wait();
    const ConvSrc<T, false> Lg{lhs, 0u}, Rg{rhs, 0u};
    acc = conv_group<D, G, T>(d, Lg, Rg, u, j, active);
  }
  if (active && j == 0) ((T*)d.out)[u_flat] = acc;
}

// EV fast path.  Block b owns vectors [b*wmul, min((b+1)*wmul, W)) of the dense p; thread 0
// keeps NSTAGE bulk copies of SVEC 32-byte vectors in flight (the "full" mbarriers complete on
// the transferred bytes), all threads consume a stage from shared memory (thread t takes
// vectors t, t+256, ...: the odometer steps +256 vectors) and each warp releases the stage on
// its "empty" mbarrier before thread 0 refills it.  Requires V*ESZ == 32 and a 32-B aligned p.
// Threads take vectors t, t+BLOCK, ...: the odometer steps +BLOCK vectors.
template <int D, int ESZ, typename IDX, int NSTAGE = TRIOT_EV_NSTAGE, int SVEC = TRIOT_EV_SVEC,
          int BLOCK = TRIOT_EV_TMA_BLOCK>
__global__ void __launch_bounds__(BLOCK) ev_tma_kernel(const __grid_constant__ Desc<IDX> d) {
  constexpr int V = 32 / ESZ;
  constexpr int NS = D + 2;
  constexpr int PER_THREAD = SVEC / BLOCK;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = (uint64_t*)(smem + (size_t)NSTAGE * SVEC * 32);
  uint64_t* empty = full + NSTAGE;
  const int tid = threadIdx.x, lane = tid & 31;
  TRIOT_TRACE(0);
  const IDX vb = (IDX)blockIdx.x * d.wmul;
  IDX ve = vb + d.wmul;
  if (ve > d.nvec || ve < vb) ve = d.nvec;
  const IDX nst = vb < ve ? (ve - vb + SVEC - 1) / SVEC : 0;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], BLOCK / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  pdl_trigger();
  pdl_wait();
  __syncthreads();
  const char* pbase = (const char*)d.t[0].ptr;
  if (tid == 0) {
    for (IDX i = 0; i < nst && i < (IDX)NSTAGE; ++i) {
      const IDX v0 = vb + i * SVEC;
      const IDX nv = (ve - v0) < (IDX)SVEC ? (ve - v0) : (IDX)SVEC;
      mbar_expect_tx(&full[i], (uint32_t)nv * 32u);
      bulk_g2s(smem + (size_t)i * SVEC * 32, pbase + (uint64_t)v0 * 32, (uint32_t)nv * 32u,
               &full[i]);
    }
  }
  IDX u[D];
  ev_decode<D, IDX>(d, vb + (IDX)tid, u);
  EvAcc<D> a;
  ev_acc_init<D, IDX>(a);
  for (IDX i = 0; i < nst; ++i) {
    const int slot = (int)(i % NSTAGE);
    const uint32_t par = (uint32_t)((i / NSTAGE) & 1);
    mbar_wait(&full[slot], par);
    if (i == 0) TRIOT_TRACE(1);
    const unsigned char* st = smem + (size_t)slot * SVEC * 32;
    const IDX v0 = vb + i * SVEC;
#pragma unroll
    for (int j = 0; j < PER_THREAD; ++j) {
      const int q = tid + j * BLOCK;
      if (v0 + (IDX)q < ve) {
        uint32_t w[8];
        const uint4 lo = *(const uint4*)(st + q * 32);
        const uint4 hi = *(const uint4*)(st + q * 32 + 16);
        w[0] = lo.x; w[1] = lo.y; w[2] = lo.z; w[3] = lo.w;
        w[4] = hi.x; w[5] = hi.y; w[6] = hi.z; w[7] = hi.w;
        ev_accumulate<D, ESZ, V, IDX>(d, w, a);
      }
      digits_step_ev<D, IDX>(d, u, a);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
    if (tid == 0 && i + NSTAGE < nst) {
      mbar_wait(&empty[slot], par);
      const IDX vn = vb + (i + NSTAGE) * SVEC;
      const IDX nv = (ve - vn) < (IDX)SVEC ? (ve - vn) : (IDX)SVEC;
      mbar_expect_tx(&full[slot], (uint32_t)nv * 32u);
      bulk_g2s(smem + (size_t)slot * SVEC * 32, pbase + (uint64_t)vn * 32, (uint32_t)nv * 32u,
               &full[slot]);
    }
  }
  TRIOT_TRACE(2);
  double acc[NS];
  ev_finish<D, IDX>(d, u, a, acc);
  ev_reduce<NS, BLOCK, IDX>(d, acc);
  TRIOT_TRACE(4);
}

}  // namespace triot
