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
