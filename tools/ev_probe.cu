// ev_probe.cu -- per-block timeline of the EV bulk-copy kernel (diagnostic tool, not product).
// Same kernel source as the library, compiled with TRIOT_EV_TRACE: thread 0 of each block
// records %globaltimer at start / first stage landed / main loop done / ticket taken / exit.
#define TRIOT_EV_TRACE 1
#include "../paper_1608_00099_b200/csrc/kernels.cuh"
#include "../paper_1608_00099_b200/csrc/plan.hpp"

#include <cstring>

using namespace triot;

extern "C" int probe_ev_c3(const double* p, double* means, void* ws, unsigned long long* trace,
                           int blocks, void* stream) {
  Geom g;
  const int64_t shape[6] = {16, 16, 16, 16, 16, 16};
  int st = plan_ev(g, p, shape, 6, 1);
  if (st) return -st;
  set_decomposition(g, 2, (uint64_t)blocks);
  unsigned grid = (unsigned)((g.nvec + g.wmul - 1) / g.wmul);
  Desc<uint32_t> d;
  memset(&d, 0, sizeof(d));
  fill_desc<uint32_t>(g, d);
  d.out = means;
  d.ws = ws;
  cudaMemcpyToSymbol(g_ev_trace, &trace, sizeof(trace));
  auto fn = ev_tma_kernel<6, 8, uint32_t>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, TRIOT_EV_SMEM);
  fn<<<grid, TRIOT_EV_TMA_BLOCK, TRIOT_EV_SMEM, (cudaStream_t)stream>>>(d);
  return cudaGetLastError() != cudaSuccess ? -100 : (int)grid;
}

// the default (LDG) kernel: chunk per warp, `bpsm` blocks per SM
extern "C" int probe_ev_ldg_c3(const double* p, double* means, void* ws, unsigned long long* trace,
                               int blocks, void* stream) {
  Geom g;
  const int64_t shape[6] = {16, 16, 16, 16, 16, 16};
  int st = plan_ev(g, p, shape, 6, 1);
  if (st) return -st;
  set_decomposition(g, 0, (uint64_t)blocks * (TRIOT_BLOCK / 32));
  const uint64_t q = g.wmul / 32, wpb = TRIOT_BLOCK / 32;
  unsigned grid = (unsigned)((g.nsteps + q * wpb - 1) / (q * wpb));
  Desc<uint32_t> d;
  memset(&d, 0, sizeof(d));
  fill_desc<uint32_t>(g, d);
  d.out = means;
  d.ws = ws;
  cudaMemcpyToSymbol(g_ev_trace, &trace, sizeof(trace));
  ev_kernel<6, 8, 4, uint32_t, 2><<<grid, TRIOT_BLOCK, 0, (cudaStream_t)stream>>>(d);
  return cudaGetLastError() != cudaSuccess ? -100 : (int)grid;
}

// variants of the LDG kernel (loads in flight K, min blocks per SM): variant index -> instance
extern "C" int probe_ev_variant_c3(const double* p, double* means, void* ws, int variant,
                                   int bpsm, void* stream) {
  Geom g;
  const int64_t shape[6] = {16, 16, 16, 16, 16, 16};
  int st = plan_ev(g, p, shape, 6, 1);
  if (st) return -st;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  set_decomposition(g, 0, (uint64_t)sms * bpsm * (TRIOT_BLOCK / 32));
  const uint64_t q = g.wmul / 32, wpb = TRIOT_BLOCK / 32;
  unsigned grid = (unsigned)((g.nsteps + q * wpb - 1) / (q * wpb));
  Desc<uint32_t> d;
  memset(&d, 0, sizeof(d));
  fill_desc<uint32_t>(g, d);
  d.out = means;
  d.ws = ws;
  static unsigned long long* scratch = nullptr;  // the kernel's trace hooks need a target
  if (!scratch && cudaMalloc(&scratch, 16384 * 8 * sizeof(unsigned long long)) != cudaSuccess)
    return -300;
  cudaMemcpyToSymbol(g_ev_trace, &scratch, sizeof(scratch));
  if (grid > 16384) return -301;
  cudaStream_t s = (cudaStream_t)stream;
  switch (variant) {
    case 0: ev_kernel<6, 8, 4, uint32_t, 2, 4><<<grid, TRIOT_BLOCK, 0, s>>>(d); break;
    case 1: ev_kernel<6, 8, 4, uint32_t, 4, 4><<<grid, TRIOT_BLOCK, 0, s>>>(d); break;
    case 2: ev_kernel<6, 8, 4, uint32_t, 4, 3><<<grid, TRIOT_BLOCK, 0, s>>>(d); break;
    case 3: ev_kernel<6, 8, 4, uint32_t, 3, 4><<<grid, TRIOT_BLOCK, 0, s>>>(d); break;
    case 4: ev_kernel<6, 8, 4, uint32_t, 8, 2><<<grid, TRIOT_BLOCK, 0, s>>>(d); break;
    case 5: ev_kernel<6, 8, 4, uint32_t, 4, 2><<<grid, TRIOT_BLOCK, 0, s>>>(d); break;
    // register-capped instances that fit more blocks per SM in one wave (48 / 40 / 32 registers)
    case 6: ev_kernel<6, 8, 4, uint32_t, 2, 5><<<grid, TRIOT_BLOCK, 0, s>>>(d); break;
    case 7: ev_kernel<6, 8, 4, uint32_t, 1, 5><<<grid, TRIOT_BLOCK, 0, s>>>(d); break;
    case 8: ev_kernel<6, 8, 4, uint32_t, 2, 6><<<grid, TRIOT_BLOCK, 0, s>>>(d); break;
    case 9: ev_kernel<6, 8, 4, uint32_t, 1, 6><<<grid, TRIOT_BLOCK, 0, s>>>(d); break;
    case 10: ev_kernel<6, 8, 4, uint32_t, 1, 8><<<grid, TRIOT_BLOCK, 0, s>>>(d); break;
    default: return -200;
  }
  return cudaGetLastError() != cudaSuccess ? -100 : (int)grid;
}

// Benchmark 2's inner product (for comparison with the EV timeline)
extern "C" int probe_dot_b2(const double* a, const double* b, double* out, void* ws,
                            unsigned long long* trace, int blocks, void* stream) {
  Geom g;
  const int64_t as[3] = {1024, 512, 256}, bs[3] = {512, 512, 32};
  int st = plan_dot(g, a, as, b, bs, nullptr, 3, 1);
  if (st) return -st;
  set_decomposition(g, 0, (uint64_t)blocks * (TRIOT_BLOCK / 32));
  const uint64_t q = g.wmul / 32, wpb = TRIOT_BLOCK / 32;
  unsigned grid = (unsigned)((g.nsteps + q * wpb - 1) / (q * wpb));
  Desc<uint32_t> d;
  memset(&d, 0, sizeof(d));
  fill_desc<uint32_t>(g, d);
  d.out = out;
  d.ws = ws;
  cudaMemcpyToSymbol(g_ev_trace, &trace, sizeof(trace));
  if (g.D != 2 || g.V != 4) return -400 - g.D * 10 - g.V;
  dot_kernel<2, 8, 4, uint32_t, 2><<<grid, TRIOT_BLOCK, 0, (cudaStream_t)stream>>>(d);
  return cudaGetLastError() != cudaSuccess ? -100 : (int)grid;
}
