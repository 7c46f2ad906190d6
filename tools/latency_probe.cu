// latency_probe.cu -- where a launch-bound op's time goes (diagnostic tool, not product): per-op
// time of 200 back-to-back launches captured in one CUDA graph, for an empty kernel with and
// without programmatic dependent launch, a one-load-one-store kernel, and the library's C1 embed
// kernel at its planned grid and at one block.  Same kernel source as the library.
#include "../paper_1608_00099_b200/csrc/kernels.cuh"
#include "../paper_1608_00099_b200/csrc/plan.hpp"

#include <cstring>

using namespace triot;

__global__ void empty_pdl() {
  pdl_trigger();
  pdl_wait();
}
__global__ void empty_plain() {}
__global__ void copy1_pdl(const double* s, double* d) {
  pdl_trigger();
  pdl_wait();
  d[threadIdx.x] = s[threadIdx.x];
}

__global__ void copy8_pdl(const double* s, double* d) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double x[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) x[j] = s[i * 4 + j];
#pragma unroll
  for (int j = 0; j < 4; ++j) d[i * 4 + j] = x[j];
}
// the same with addresses formed from many fields of the 1.3 KB descriptor (constant bank)
__global__ void copy8_desc_pdl(const __grid_constant__ Desc<uint32_t> d) {
  uint32_t o = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) o += d.ext[k] * d.t[0].sig[k] + d.fdm[k] + d.t[1].kap[k];
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const double* s = (const double*)d.t[1].ptr;
  double* q = (double*)d.t[0].ptr;
  double x[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) x[j] = s[(i * 4 + j + o) & 1023];
#pragma unroll
  for (int j = 0; j < 4; ++j) q[i * 4 + j] = x[j];
}

// 64 KB moved as one 32-byte vector per thread, any block size (what is the floor of C1's
// bytes, and does the block shape matter?); mode 1 = stores only, 2 = loads only
__global__ void copyv_pdl(const double* s, double* d, int mode) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (mode != 1) Mem<32>::ld(s + 4 * i, w);
  if (mode != 2) Mem<32>::st(d + 4 * i, w);
  else if (w[0] == 0x12345u) d[0] = 1.0;
}

static int launch(const void* fn, unsigned grid, unsigned block, void** args, cudaStream_t st,
                  bool pdl) {
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return (int)cudaLaunchKernelExC(&cfg, fn, args);
}

// variant: 0 empty+pdl, 1 empty plain, 2 copy1+pdl, 3 C1 embed planned grid, 4 C1 embed 1 block,
// 5 C1 embed planned grid without PDL.  Returns us per op (graph of n launches, 5 replays).
extern "C" double probe_latency(int variant, void* dst, const void* src, void* scratch, int n) {
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  Geom g;
  const int64_t dsh[4] = {8, 16, 8, 8}, ssh[4] = {4, 9, 7, 5};
  plan_embed(g, dst, dsh, src, ssh, 4, 1, 0);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned grid = variant == 4 ? 1u : 8u;
  const unsigned eblock = (unsigned)TRIOT_BLOCK;
  set_decomposition(g, 0, (uint64_t)grid * (eblock / 32));
  Desc<uint32_t> d;
  memset(&d, 0, sizeof(d));
  fill_desc<uint32_t>(g, d);
  const void* efn = (const void*)&embed_kernel<4, 8, 4, uint32_t, 4, false>;
  // a small product of two PMFs of different shapes (64 KB out): c (8,16,8,8) = a (9,16,8,8) * b (8,17,8,8)
  Geom gb;
  const int64_t ash[4] = {9, 16, 8, 8}, bsh[4] = {8, 17, 8, 8};
  const char* sc = (const char*)scratch;
  plan_binary(gb, (void*)dst, dsh, sc, ash, sc + 9 * 16 * 64 * 8, bsh, dsh, 4, 1, 2);
  set_decomposition(gb, 0, (uint64_t)8 * (TRIOT_BLOCK / 32));
  Desc<uint32_t> db;
  memset(&db, 0, sizeof(db));
  fill_desc<uint32_t>(gb, db);
  const void* bfn = gb.D == 2   ? (const void*)&binary_kernel<2, 8, 4, uint32_t, 2, 2>
                    : gb.D == 3 ? (const void*)&binary_kernel<3, 8, 4, uint32_t, 2, 2>
                                : (const void*)&binary_kernel<4, 8, 4, uint32_t, 2, 2>;
  void* bargs[1] = {&db};
  if (variant == 9 && (gb.V != 4 || gb.D < 2 || gb.D > 4)) return -2.0;
  void* eargs[1] = {&d};
  const double* s = (const double*)scratch;
  double* o = (double*)scratch + 8192;
  void* cargs[2] = {&s, &o};
  int cmode = variant == 14 ? 1 : variant == 15 ? 2 : 0;
  void* vargs[3] = {&s, &o, &cmode};
  const unsigned vblock = variant == 10 ? 256 : variant == 11 ? 128 : variant == 12 ? 64 : variant == 13 ? 32 : 256;
  cudaGraph_t gr;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < n; ++i) {
    switch (variant) {
      case 0: launch((const void*)empty_pdl, 1, 32, nullptr, st, true); break;
      case 1: launch((const void*)empty_plain, 1, 32, nullptr, st, false); break;
      case 2: launch((const void*)copy1_pdl, 1, 32, cargs, st, true); break;
      case 3: case 4: launch(efn, grid, eblock, eargs, st, true); break;
      case 6: launch((const void*)copy8_pdl, 8, 256, cargs, st, true); break;
      case 9: launch(bfn, 8, TRIOT_BLOCK, bargs, st, true); break;
      case 7: launch((const void*)copy8_desc_pdl, 8, 256, eargs, st, true); break;
      case 10: case 11: case 12: case 13: case 14: case 15:
        launch((const void*)copyv_pdl, 2048 / vblock, vblock, vargs, st, true); break;
      default: launch(efn, grid, TRIOT_BLOCK, eargs, st, false); break;
    }
  }
  cudaStreamEndCapture(st, &gr);
  if (cudaGraphInstantiate(&ge, gr, 0) != cudaSuccess) return -1;
  cudaGraphLaunch(ge, st);
  cudaStreamSynchronize(st);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, st);
  for (int r = 0; r < 5; ++r) cudaGraphLaunch(ge, st);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(gr);
  cudaStreamDestroy(st);
  return ms * 1000.0 / (5.0 * n);
}
