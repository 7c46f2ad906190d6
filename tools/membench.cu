// membench.cu -- HBM ceilings for the traffic mixes of the TRIOT ops (diagnostic tool, not product).
// Pure write / pure read / copy / read-fraction mixes with 256-bit accesses, contiguous
// per-warp chunks (the same decomposition as the product kernels), several store policies.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC -o libmembench.so membench.cu
#include <cuda_runtime.h>
#include <stdint.h>

template <int POL>
__device__ __forceinline__ void st256(void* p, uint32_t a, uint32_t b) {
  if (POL == 0)
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%1,%2,%1,%2,%1,%2};" ::"l"(p), "r"(a), "r"(b) : "memory");
  else if (POL == 1)
    asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1,%2,%1,%2,%1,%2,%1,%2};" ::"l"(p), "r"(a), "r"(b) : "memory");
  else if (POL == 2)
    asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%1,%2,%1,%2,%1,%2};" ::"l"(p), "r"(a), "r"(b) : "memory");
  else
    asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%2,%1,%2,%1,%2,%1,%2};" ::"l"(p), "r"(a), "r"(b) : "memory");
}

struct alignas(32) W8 { uint32_t w[8]; };

__device__ __forceinline__ W8 ld256(const void* p) {
  W8 r;
  asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]),
                 "=r"(r.w[5]), "=r"(r.w[6]), "=r"(r.w[7])
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st256v(void* p, const W8& r) {
  asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p),
               "r"(r.w[0]), "r"(r.w[1]), "r"(r.w[2]), "r"(r.w[3]), "r"(r.w[4]), "r"(r.w[5]),
               "r"(r.w[6]), "r"(r.w[7])
               : "memory");
}

// n32: number of 32-byte vectors; each warp owns a contiguous chunk of q steps of 32 vectors
template <int POL, int U>
__global__ void write_k(char* dst, uint64_t n32, uint64_t q) {
  uint64_t warp = (uint64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  uint64_t lane = threadIdx.x & 31;
  uint64_t s0 = warp * q, s1 = s0 + q;
  for (uint64_t s = s0; s < s1; s += U) {
#pragma unroll
    for (int j = 0; j < U; ++j) {
      uint64_t v = (s + j) * 32 + lane;
      if (s + j < s1 && v < n32) st256<POL>(dst + v * 32, 0u, 0u);
    }
  }
}

template <int U>
__global__ void read_k(const char* src, uint64_t n32, uint64_t q, uint32_t* sink) {
  uint64_t warp = (uint64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  uint64_t lane = threadIdx.x & 31;
  uint64_t s0 = warp * q, s1 = s0 + q;
  uint32_t acc = 0;
  for (uint64_t s = s0; s < s1; s += U) {
    W8 r[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      uint64_t v = (s + j) * 32 + lane;
      if (s + j < s1 && v < n32) r[j] = ld256(src + v * 32);
      else r[j] = W8{};
    }
#pragma unroll
    for (int j = 0; j < U; ++j)
#pragma unroll
      for (int k = 0; k < 8; ++k) acc ^= r[j].w[k];
  }
  if (acc == 0x9e3779b9u) sink[0] = acc;
}

// read `rd_pct`% of the vectors (a leading part of every 32-vector group... per step mask) and
// write all: the embed mix (C2 ~ 42 % of the dst vectors read).
template <int U>
__global__ void mix_k(const char* src, char* dst, uint64_t n32, uint64_t q, uint32_t rd_of_64) {
  uint64_t warp = (uint64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  uint64_t lane = threadIdx.x & 31;
  uint64_t s0 = warp * q, s1 = s0 + q;
  for (uint64_t s = s0; s < s1; s += U) {
    W8 r[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      uint64_t v = (s + j) * 32 + lane;
      bool rd = (v & 63) < rd_of_64;
      if (s + j < s1 && v < n32 && rd) r[j] = ld256(src + v * 32);
      else r[j] = W8{};
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      uint64_t v = (s + j) * 32 + lane;
      if (s + j < s1 && v < n32) st256v(dst + v * 32, r[j]);
    }
  }
}

static void geom(uint64_t n32, int blocks, int threads, uint64_t* q) {
  uint64_t warps = (uint64_t)blocks * (threads / 32);
  uint64_t steps = (n32 + 31) / 32;
  *q = (steps + warps - 1) / warps;
}

extern "C" int mb_write(void* dst, uint64_t bytes, int blocks, int threads, int pol, int u,
                        void* stream) {
  uint64_t n32 = bytes / 32, q;
  geom(n32, blocks, threads, &q);
  cudaStream_t s = (cudaStream_t)stream;
#define W(P, UU) write_k<P, UU><<<blocks, threads, 0, s>>>((char*)dst, n32, q)
  if (u == 4) {
    if (pol == 0) W(0, 4); else if (pol == 1) W(1, 4); else if (pol == 2) W(2, 4); else W(3, 4);
  } else if (u == 8) {
    if (pol == 0) W(0, 8); else if (pol == 1) W(1, 8); else if (pol == 2) W(2, 8); else W(3, 8);
  } else {
    if (pol == 0) W(0, 1); else if (pol == 1) W(1, 1); else if (pol == 2) W(2, 1); else W(3, 1);
  }
  return (int)cudaGetLastError();
}

extern "C" int mb_read(const void* src, uint64_t bytes, int blocks, int threads, int u,
                       void* sink, void* stream) {
  uint64_t n32 = bytes / 32, q;
  geom(n32, blocks, threads, &q);
  cudaStream_t s = (cudaStream_t)stream;
  if (u == 8) read_k<8><<<blocks, threads, 0, s>>>((const char*)src, n32, q, (uint32_t*)sink);
  else if (u == 2) read_k<2><<<blocks, threads, 0, s>>>((const char*)src, n32, q, (uint32_t*)sink);
  else read_k<4><<<blocks, threads, 0, s>>>((const char*)src, n32, q, (uint32_t*)sink);
  return (int)cudaGetLastError();
}

extern "C" int mb_mix(const void* src, void* dst, uint64_t bytes, int blocks, int threads, int u,
                      int rd_of_64, void* stream) {
  uint64_t n32 = bytes / 32, q;
  geom(n32, blocks, threads, &q);
  cudaStream_t s = (cudaStream_t)stream;
  if (u == 8) mix_k<8><<<blocks, threads, 0, s>>>((const char*)src, (char*)dst, n32, q, rd_of_64);
  else if (u == 2) mix_k<2><<<blocks, threads, 0, s>>>((const char*)src, (char*)dst, n32, q, rd_of_64);
  else mix_k<4><<<blocks, threads, 0, s>>>((const char*)src, (char*)dst, n32, q, rd_of_64);
  return (int)cudaGetLastError();
}

// grid-stride variants: at any moment all warps work inside one window of the buffer
template <int POL, int U>
__global__ void write_gs(char* dst, uint64_t n32) {
  uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t T = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = tid; base < n32; base += T * U) {
#pragma unroll
    for (int j = 0; j < U; ++j) {
      uint64_t v = base + j * T;
      if (v < n32) st256<POL>(dst + v * 32, 0u, 0u);
    }
  }
}
template <int U>
__global__ void mix_gs(const char* src, char* dst, uint64_t n32, uint32_t rd_of_64) {
  uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t T = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = tid; base < n32; base += T * U) {
    W8 r[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      uint64_t v = base + j * T;
      if (v < n32 && (v & 63) < rd_of_64) r[j] = ld256(src + v * 32);
      else r[j] = W8{};
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      uint64_t v = base + j * T;
      if (v < n32) st256v(dst + v * 32, r[j]);
    }
  }
}
// block-chunk variant: block b owns a contiguous chunk; inside it the warps interleave
template <int U>
__global__ void mix_bc(const char* src, char* dst, uint64_t n32, uint64_t per_block, uint32_t rd_of_64) {
  uint64_t b0 = (uint64_t)blockIdx.x * per_block, b1 = b0 + per_block;
  if (b1 > n32) b1 = n32;
  for (uint64_t base = b0 + threadIdx.x; base < b1; base += (uint64_t)blockDim.x * U) {
    W8 r[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      uint64_t v = base + j * blockDim.x;
      if (v < b1 && (v & 63) < rd_of_64) r[j] = ld256(src + v * 32);
      else r[j] = W8{};
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      uint64_t v = base + j * blockDim.x;
      if (v < b1) st256v(dst + v * 32, r[j]);
    }
  }
}

extern "C" int mb_write_gs(void* dst, uint64_t bytes, int blocks, int threads, int pol, int u, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  uint64_t n32 = bytes / 32;
  if (u == 4) { if (pol == 0) write_gs<0,4><<<blocks,threads,0,s>>>((char*)dst,n32); else write_gs<2,4><<<blocks,threads,0,s>>>((char*)dst,n32); }
  else { if (pol == 0) write_gs<0,1><<<blocks,threads,0,s>>>((char*)dst,n32); else write_gs<2,1><<<blocks,threads,0,s>>>((char*)dst,n32); }
  return (int)cudaGetLastError();
}
extern "C" int mb_mix_gs(const void* src, void* dst, uint64_t bytes, int blocks, int threads, int u, int rd, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  uint64_t n32 = bytes / 32;
  if (u == 4) mix_gs<4><<<blocks,threads,0,s>>>((const char*)src,(char*)dst,n32,rd);
  else if (u == 2) mix_gs<2><<<blocks,threads,0,s>>>((const char*)src,(char*)dst,n32,rd);
  else mix_gs<1><<<blocks,threads,0,s>>>((const char*)src,(char*)dst,n32,rd);
  return (int)cudaGetLastError();
}
extern "C" int mb_mix_bc(const void* src, void* dst, uint64_t bytes, int blocks, int threads, int u, int rd, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  uint64_t n32 = bytes / 32;
  uint64_t per = (n32 + blocks - 1) / blocks;
  if (u == 4) mix_bc<4><<<blocks,threads,0,s>>>((const char*)src,(char*)dst,n32,per,rd);
  else mix_bc<2><<<blocks,threads,0,s>>>((const char*)src,(char*)dst,n32,per,rd);
  return (int)cudaGetLastError();
}

// one-shot grid (the shape of torch's elementwise kernels): block b writes blockDim*U vectors of
// VB bytes starting at b*blockDim*U*VB, interleaved by thread; every thread exits after U stores
template <int VB, int U>
__global__ void write_os(char* dst, uint64_t nv) {
  uint64_t base = (uint64_t)blockIdx.x * blockDim.x * U + threadIdx.x;
#pragma unroll
  for (int j = 0; j < U; ++j) {
    uint64_t v = base + (uint64_t)j * blockDim.x;
    if (v < nv) {
      if (VB == 32) st256<1>(dst + v * 32, 0u, 0u);
      else asm volatile("st.global.v4.b32 [%0], {%1,%1,%1,%1};" ::"l"(dst + v * 16), "r"(0u) : "memory");
    }
  }
}
extern "C" int mb_write_os(void* dst, uint64_t bytes, int vb, int threads, int u, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  uint64_t nv = bytes / vb;
  uint64_t per = (uint64_t)threads * u;
  unsigned blocks = (unsigned)((nv + per - 1) / per);
#define OS(VB_, U_) write_os<VB_, U_><<<blocks, threads, 0, s>>>((char*)dst, nv)
  if (vb == 32) { if (u == 1) OS(32, 1); else if (u == 2) OS(32, 2); else if (u == 4) OS(32, 4); else OS(32, 8); }
  else { if (u == 1) OS(16, 1); else if (u == 2) OS(16, 2); else if (u == 4) OS(16, 4); else OS(16, 8); }
  return (int)cudaGetLastError();
}

// one-shot read: block b reads blockDim*U 32-B vectors starting at b*blockDim*U, interleaved by
// thread, folds them and writes one word per block (the shape of a one-partial-per-block
// reduction)
template <int U>
__global__ void read_os(const char* src, uint64_t nv, uint32_t* part) {
  uint64_t base = (uint64_t)blockIdx.x * blockDim.x * U + threadIdx.x;
  W8 r[U];
#pragma unroll
  for (int j = 0; j < U; ++j) {
    uint64_t v = base + (uint64_t)j * blockDim.x;
    if (v < nv) r[j] = ld256(src + v * 32); else r[j] = W8{};
  }
  uint32_t acc = 0;
#pragma unroll
  for (int j = 0; j < U; ++j)
#pragma unroll
    for (int k = 0; k < 8; ++k) acc ^= r[j].w[k];
  acc = __reduce_xor_sync(0xffffffffu, acc);
  if ((threadIdx.x & 31) == 0) atomicXor(part + blockIdx.x, acc);
}
extern "C" int mb_read_os(const void* src, uint64_t bytes, int threads, int u, void* part, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  uint64_t nv = bytes / 32, per = (uint64_t)threads * u;
  unsigned blocks = (unsigned)((nv + per - 1) / per);
#define ROS(U_) read_os<U_><<<blocks, threads, 0, s>>>((const char*)src, nv, (uint32_t*)part)
  if (u == 1) ROS(1); else if (u == 2) ROS(2); else if (u == 4) ROS(4); else if (u == 8) ROS(8); else ROS(16);
  return (int)cudaGetLastError();
}

// write_k<pol 1, U 4> with occupancy limited by dynamic shared memory (blocks per SM)
extern "C" int mb_write_occ(void* dst, uint64_t bytes, int blocks, int threads, int smem, void* stream) {
  uint64_t n32 = bytes / 32, q;
  geom(n32, blocks, threads, &q);
  cudaStream_t s = (cudaStream_t)stream;
  if (smem > 48 * 1024) cudaFuncSetAttribute(write_k<1, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  write_k<1, 4><<<blocks, threads, smem, s>>>((char*)dst, n32, q);
  return (int)cudaGetLastError();
}
