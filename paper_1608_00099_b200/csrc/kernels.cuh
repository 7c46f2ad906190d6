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
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "desc.h"

namespace triot {

constexpr int kBlock = TRIOT_BLOCK;

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
  static __device__ __forceinline__ void st(void* p, const uint32_t* w) {
    asm volatile("st.global.v2.b32 [%0], {%1,%2};" ::"l"(p), "r"(w[0]), "r"(w[1]) : "memory");
  }
};
template <>
struct Mem<4> {
  static __device__ __forceinline__ void ld(const void* p, uint32_t* w) {
    asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(w[0]) : "l"(p));
  }
  static __device__ __forceinline__ void st(void* p, const uint32_t* w) {
    asm volatile("st.global.b32 [%0], %1;" ::"l"(p), "r"(w[0]) : "memory");
  }
};

template <int ESZ, typename IDX>
__device__ __forceinline__ const char* addr(const void* base, IDX off) {
  return (const char*)base + (uint64_t)off * ESZ;
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

// Decode vector index v into digits, then Horner offsets per tensor (Alg 2).
template <int D, int NT, bool BOUNDS, typename IDX>
__device__ __forceinline__ void odo_start(const Desc<IDX>& d, IDX v, IDX (&u)[D],
                                          IDX (&off)[NT], uint32_t& oob) {
#pragma unroll
  for (int k = D - 1; k >= 1; --k) {
    IDX q = divq<IDX>(v, d.ext[k], d.fdm[k], d.fds[k]);
    u[k] = v - q * d.ext[k];
    v = q;
  }
  u[0] = v;
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
template <int D, int NT, bool BOUNDS, typename IDX>
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
    if (BOUNDS && k < D - 1) oob = (oob & ~(1u << k)) | ((uint32_t)(nu >= d.bnd[k]) << k);
    if (k <= d.klo && !carry) break;  // "No more carry operations" (Alg 3)
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

template <int ESZ, int V, typename IDX>
__device__ __forceinline__ void load_vec(const TensorAcc<IDX>& t, IDX off, uint32_t lgL,
                                         uint32_t* w) {
  constexpr int EW = ESZ / 4;
  if (V > 1 && t.vec) {
    Mem<V * ESZ>::ld(addr<ESZ>(t.ptr, off), w);
  } else {
#pragma unroll
    for (int e = 0; e < V; ++e) Mem<ESZ>::ld(addr<ESZ>(t.ptr, elem_off(off, e, lgL, t.rho, t.tau)), w + e * EW);
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

template <int D, int ESZ, int V, typename IDX, int K>
__global__ void __launch_bounds__(kBlock) embed_kernel(const __grid_constant__ Desc<IDX> d) {
  constexpr int EW = ESZ / 4;
  constexpr int NW = V * EW;
  const int lane = threadIdx.x & 31;
  const IDX warp = (IDX)blockIdx.x * (kBlock / 32) + (IDX)(threadIdx.x >> 5);
  const IDX base0 = warp * d.wmul;
  if (base0 >= d.nvec) return;
  const IDX vend = warp_end(d, base0);
  IDX u[D], off[2];
  uint32_t oob;
  IDX v = base0 + (IDX)lane;
  odo_start<D, 2, true, IDX>(d, v, u, off, oob);
  const uint32_t lgL = d.lgL;
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
      odo_step<D, 2, true, IDX>(d, u, off, oob);
    }
#pragma unroll
    for (int j = 0; j < K; ++j)
      if (valid[j]) store_vec<ESZ, V, IDX>(d.t[0], doff[j], lgL, buf[j]);
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
  if (base0 >= d.nvec) return;
  const IDX vend = warp_end(d, base0);
  IDX u[D], off[3];
  uint32_t oob;
  IDX v = base0 + (IDX)lane;
  odo_start<D, 3, false, IDX>(d, v, u, off, oob);
  const uint32_t lgL = d.lgL;
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
        load_vec<ESZ, V, IDX>(d.t[1], off[1], lgL, ba[j]);
        load_vec<ESZ, V, IDX>(d.t[2], off[2], lgL, bb[j]);
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

// ------------------------------------------------------------------ expected value
// m_k = sum_t t_k p[t] (Alg 11) in fp64.  Per vector the outer digits are constant,
// so with s = sum_e p_e:  acc_k += u_k * s (outer digits) and the vector digit contributes
// (first row/col) * s plus the small in-vector weights.  Per-lane accumulators, then a
// fixed-order warp butterfly, fixed-order cross-warp sum, one partial per block, and the last
// block (ticket) sums the partials in a fixed order: deterministic run to run ("each thread
// computes its own pre-result and these pre-results are amalgamated").

template <int D, int ESZ, int V, typename IDX, int K>
__global__ void __launch_bounds__(kBlock) ev_kernel(const __grid_constant__ Desc<IDX> d) {
  constexpr int EW = ESZ / 4;
  constexpr int NW = V * EW;
  constexpr int NS = D + 1;  // weight slots (D digits + the column slot of a collapsed vector)
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const IDX warp = (IDX)blockIdx.x * (kBlock / 32) + (IDX)wib;
  const IDX base0 = warp * d.wmul;
  double acc[NS];
#pragma unroll
  for (int k = 0; k < NS; ++k) acc[k] = 0.0;
  const uint32_t lgL = d.lgL;
  if (base0 < d.nvec) {
    const IDX vend = warp_end(d, base0);
    IDX u[D], off[1];
    uint32_t oob;
    IDX v = base0 + (IDX)lane;
    odo_start<D, 1, false, IDX>(d, v, u, off, oob);
    const IDX vmul = d.rowmul + d.colmul;  // exactly one of them is nonzero
    const bool coll = d.collapsed != 0;
    for (IDX b = base0; b < vend; b += K * d.dv) {
      uint32_t buf[K][NW];
      bool valid[K];
      IDX uu[K][D];
#pragma unroll
      for (int j = 0; j < K; ++j) {
        valid[j] = v < vend;
        v += d.dv;
        if (valid[j]) load_vec<ESZ, V, IDX>(d.t[0], off[0], lgL, buf[j]);
#pragma unroll
        for (int k = 0; k < D; ++k) uu[j][k] = u[k];
        odo_step<D, 1, false, IDX>(d, u, off, oob);
      }
#pragma unroll
      for (int j = 0; j < K; ++j) {
        if (!valid[j]) continue;
        double x[V];
#pragma unroll
        for (int e = 0; e < V; ++e) x[e] = (double)Elem<ESZ>::get(buf[j] + e * EW);
        double sum = x[0];
#pragma unroll
        for (int e = 1; e < V; ++e) sum += x[e];
        double wr = 0.0, wc = 0.0;
#pragma unroll
        for (int e = 1; e < V; ++e) {
          wr = fma((double)((uint32_t)e >> lgL), x[e], wr);
          wc = fma((double)((uint32_t)e & ((1u << lgL) - 1u)), x[e], wc);
        }
#pragma unroll
        for (int k = 0; k < D - 1; ++k) acc[k] = fma((double)uu[j][k], sum, acc[k]);
        acc[D - 1] += fma((double)(uu[j][D - 1] * vmul), sum, coll ? wr : wc);
        if (coll) acc[D] += wc;
      }
    }
  }
  // ---- deterministic reduction
#pragma unroll
  for (int k = 0; k < NS; ++k) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
  }
  __shared__ double sm[kBlock / 32][NS];
  __shared__ int is_last;
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NS; ++k) sm[wib][k] = acc[k];
  }
  __syncthreads();
  unsigned* ticket = (unsigned*)d.ws;
  double* part = (double*)((char*)d.ws + TRIOT_EV_WS_HEADER);
  if (threadIdx.x < NS) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < kBlock / 32; ++w) t += sm[w][threadIdx.x];
    part[(size_t)blockIdx.x * NS + threadIdx.x] = t;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  double f[NS];
#pragma unroll
  for (int k = 0; k < NS; ++k) f[k] = 0.0;
  for (unsigned b = threadIdx.x; b < gridDim.x; b += kBlock) {
#pragma unroll
    for (int k = 0; k < NS; ++k) f[k] += __ldcg(part + (size_t)b * NS + k);
  }
#pragma unroll
  for (int k = 0; k < NS; ++k) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) f[k] += __shfl_xor_sync(0xffffffffu, f[k], o);
  }
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NS; ++k) sm[wib][k] = f[k];
  }
  __syncthreads();
  __shared__ double tot[NS];
  if (threadIdx.x < NS) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < kBlock / 32; ++w) t += sm[w][threadIdx.x];
    tot[threadIdx.x] = t;
  }
  __syncthreads();
  if (threadIdx.x < (unsigned)d.d_out) {
    const int sl = d.slot_of_axis[threadIdx.x];
    ((double*)d.out)[threadIdx.x] = sl >= 0 ? tot[sl] : 0.0;
  }
  if (threadIdx.x == 0) *ticket = 0u;  // leave the workspace ready for the next call
}

}  // namespace triot
