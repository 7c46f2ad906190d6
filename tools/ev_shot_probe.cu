// ev_shot_probe.cu -- variants of the one-shot expected-value kernel on C3 (diagnostic tool,
// not product): loads per thread J x min blocks per SM, grid cap; same kernel source as the
// library.  Built by tools/ev_shot_probe.py.
#include "../paper_1608_00099_b200/csrc/kernels.cuh"
#include "../paper_1608_00099_b200/csrc/plan.hpp"

#include <cstring>

using namespace triot;

template <int J, int MINB>
static int go(const Desc<uint32_t>& d, unsigned grid, cudaStream_t s) {
  ev_shot_kernel<6, 8, 4, uint32_t, J, MINB><<<grid, TRIOT_BLOCK, 0, s>>>(d);
  return 0;
}

static const int kJ[] = {1, 2, 2, 4, 4, 2, 8, 1, 4};
static const int kMinb[] = {8, 8, 6, 4, 6, 4, 2, 6, 3};

extern "C" int probe_variants(void) { return (int)(sizeof(kJ) / sizeof(kJ[0])); }
extern "C" int probe_variant_info(int v, int* j, int* minb, int* regs) {
  const void* fns[] = {
      (const void*)ev_shot_kernel<6, 8, 4, uint32_t, 1, 8>, (const void*)ev_shot_kernel<6, 8, 4, uint32_t, 2, 8>,
      (const void*)ev_shot_kernel<6, 8, 4, uint32_t, 2, 6>, (const void*)ev_shot_kernel<6, 8, 4, uint32_t, 4, 4>,
      (const void*)ev_shot_kernel<6, 8, 4, uint32_t, 4, 6>, (const void*)ev_shot_kernel<6, 8, 4, uint32_t, 2, 4>,
      (const void*)ev_shot_kernel<6, 8, 4, uint32_t, 8, 2>, (const void*)ev_shot_kernel<6, 8, 4, uint32_t, 1, 6>,
      (const void*)ev_shot_kernel<6, 8, 4, uint32_t, 4, 3>};
  cudaFuncAttributes a;
  if (cudaFuncGetAttributes(&a, fns[v]) != cudaSuccess) return -1;
  *j = kJ[v];
  *minb = kMinb[v];
  *regs = a.numRegs;
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fns[v], TRIOT_BLOCK, 0);
  return nb;
}

// variant v, grid = min(units, gridcap) (gridcap 0: all units)
extern "C" int probe_shot_c3(const double* p, double* means, void* ws, int v, int gridcap,
                             void* stream) {
  Geom g;
  const int64_t shape[6] = {16, 16, 16, 16, 16, 16};
  int st = plan_ev(g, p, shape, 6, 1);
  if (st) return -st;
  const uint64_t unit = (uint64_t)TRIOT_BLOCK * kJ[v];
  uint64_t grid = (g.nvec + unit - 1) / unit;
  if (gridcap > 0 && grid > (uint64_t)gridcap) grid = gridcap;
  if (grid > TRIOT_EV_MAX_GRID) grid = TRIOT_EV_MAX_GRID;
  uint32_t G = TRIOT_EV_MIN_GROUP;
  while ((uint64_t)G * G < grid) G <<= 1;
  g.rgroup = G;
  Desc<uint32_t> d;
  memset(&d, 0, sizeof(d));
  fill_desc<uint32_t>(g, d);
  d.out = means;
  d.ws = ws;
  cudaStream_t s = (cudaStream_t)stream;
  switch (v) {
    case 0: go<1, 8>(d, grid, s); break;
    case 1: go<2, 8>(d, grid, s); break;
    case 2: go<2, 6>(d, grid, s); break;
    case 3: go<4, 4>(d, grid, s); break;
    case 4: go<4, 6>(d, grid, s); break;
    case 5: go<2, 4>(d, grid, s); break;
    case 6: go<8, 2>(d, grid, s); break;
    case 7: go<1, 6>(d, grid, s); break;
    case 8: go<4, 3>(d, grid, s); break;
    default: return -200;
  }
  return cudaGetLastError() != cudaSuccess ? -100 : (int)grid;
}

// ---- ev_dyn_kernel variants: (J, B) ring; R rounds per unit (0: the fewest that keep the
// unit partials within one final batch); grid = SMs (or gridcap)
static const int kDJ[] = {1, 1, 2, 1, 2};
static const int kDB[] = {2, 3, 2, 4, 3};
extern "C" int probe_dyn_variants(void) { return (int)(sizeof(kDJ) / sizeof(kDJ[0])); }
extern "C" int probe_dyn_info(int v, int* j, int* b, int* regs) {
  const void* fns[] = {(const void*)ev_dyn_kernel<6, 8, 4, uint32_t, 1, 2>,
                       (const void*)ev_dyn_kernel<6, 8, 4, uint32_t, 1, 3>,
                       (const void*)ev_dyn_kernel<6, 8, 4, uint32_t, 2, 2>,
                       (const void*)ev_dyn_kernel<6, 8, 4, uint32_t, 1, 4>,
                       (const void*)ev_dyn_kernel<6, 8, 4, uint32_t, 2, 3>};
  cudaFuncAttributes a;
  if (cudaFuncGetAttributes(&a, fns[v]) != cudaSuccess) return -1;
  *j = kDJ[v];
  *b = kDB[v];
  *regs = a.numRegs;
  return a.localSizeBytes;
}
extern "C" int probe_dyn_c3(const double* p, double* means, void* ws, int v, int rforce,
                            int gridcap, void* stream) {
  Geom g;
  const int64_t shape[6] = {16, 16, 16, 16, 16, 16};
  int st = plan_ev(g, p, shape, 6, 1);
  if (st) return -st;
  const uint64_t rv = (uint64_t)kDyn * kDJ[v];
  const uint64_t nrounds = (g.nvec + rv - 1) / rv;
  const uint64_t maxu = kDynFinalDoubles / ev_slot_pad(8);
  uint64_t R = (nrounds + maxu - 1) / maxu;
  if (rforce > 0 && (uint64_t)rforce > R) R = rforce;
  const uint64_t nu = (nrounds + R - 1) / R;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint64_t grid = gridcap > 0 ? (uint64_t)gridcap : (uint64_t)sms;
  if (grid > nu) grid = nu;
  g.wmul = R;
  g.wspan = nu;
  Desc<uint32_t> d;
  memset(&d, 0, sizeof(d));
  fill_desc<uint32_t>(g, d);
  d.out = means;
  d.ws = ws;
  cudaStream_t s = (cudaStream_t)stream;
  switch (v) {
    case 0: ev_dyn_kernel<6, 8, 4, uint32_t, 1, 2><<<grid, kDyn, 0, s>>>(d); break;
    case 1: ev_dyn_kernel<6, 8, 4, uint32_t, 1, 3><<<grid, kDyn, 0, s>>>(d); break;
    case 2: ev_dyn_kernel<6, 8, 4, uint32_t, 2, 2><<<grid, kDyn, 0, s>>>(d); break;
    case 3: ev_dyn_kernel<6, 8, 4, uint32_t, 1, 4><<<grid, kDyn, 0, s>>>(d); break;
    case 4: ev_dyn_kernel<6, 8, 4, uint32_t, 2, 3><<<grid, kDyn, 0, s>>>(d); break;
    default: return -200;
  }
  return cudaGetLastError() != cudaSuccess ? -100 : (int)(grid * 100000 + nu);
}

// ---- ev_fx_kernel variants: K loads per lane per unit; grid = SMs x blocks per SM (occupancy)
static const int kFK[] = {4, 8, 4, 8};
extern "C" int probe_fx_variants(void) { return 4; }
static const void* fx_fn(int v) {
  switch (v) {
    case 0: return (const void*)ev_fx_kernel<6, 8, 4, uint32_t, 4>;
    case 1: return (const void*)ev_fx_kernel<6, 8, 4, uint32_t, 8>;
    case 2: return (const void*)ev_fx_kernel<6, 8, 4, uint32_t, 4, 0>;
    default: return (const void*)ev_fx_kernel<6, 8, 4, uint32_t, 8, 0>;
  }
}
extern "C" int probe_fx_info(int v, int* k, int* regs, int* occ) {
  const void* fn = fx_fn(v);
  const int smem = kFxWarps * 8 * kFxNL * 8;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncAttributes a;
  if (cudaFuncGetAttributes(&a, fn) != cudaSuccess) return -1;
  *k = kFK[v];
  *regs = a.numRegs;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, fn, kFxBlock, smem);
  return a.localSizeBytes;
}
extern "C" int probe_fx_c3(const double* p, double* means, void* ws, int v, int bpsm,
                           void* stream) {
  Geom g;
  const int64_t shape[6] = {16, 16, 16, 16, 16, 16};
  int st = plan_ev(g, p, shape, 6, 1);
  if (st) return -st;
  set_decomposition(g, 0, 1);  // +32-vector step digits
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = kFxWarps * 8 * kFxNL * 8;
  const void* fn = fx_fn(v);
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned grid = (unsigned)(sms * bpsm);
  Desc<uint32_t> d;
  memset(&d, 0, sizeof(d));
  fill_desc<uint32_t>(g, d);
  d.out = means;
  d.ws = ws;
  cudaStream_t s = (cudaStream_t)stream;
  switch (v) {
    case 0: ev_fx_kernel<6, 8, 4, uint32_t, 4><<<grid, kFxBlock, smem, s>>>(d); break;
    case 1: ev_fx_kernel<6, 8, 4, uint32_t, 8><<<grid, kFxBlock, smem, s>>>(d); break;
    case 2: ev_fx_kernel<6, 8, 4, uint32_t, 4, 0><<<grid, kFxBlock, smem, s>>>(d); break;
    default: ev_fx_kernel<6, 8, 4, uint32_t, 8, 0><<<grid, kFxBlock, smem, s>>>(d); break;
  }
  return cudaGetLastError() != cudaSuccess ? -100 : (int)grid;
}

// ---- the library's ev_kernel (chunk per warp, telescoped) at `bpsm` blocks per SM
extern "C" int probe_evk_c3(const double* p, double* means, void* ws, int bpsm, void* stream) {
  Geom g;
  const int64_t shape[6] = {16, 16, 16, 16, 16, 16};
  int st = plan_ev(g, p, shape, 6, 1);
  if (st) return -st;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  set_decomposition(g, 0, (uint64_t)sms * bpsm * (TRIOT_BLOCK / 32));
  const uint64_t q = g.wmul / 32, wpb = TRIOT_BLOCK / 32;
  unsigned grid = (unsigned)((g.nsteps + q * wpb - 1) / (q * wpb));
  uint32_t G = TRIOT_EV_MIN_GROUP;
  while ((uint64_t)G * G < grid) G <<= 1;
  g.rgroup = G;
  Desc<uint32_t> d;
  memset(&d, 0, sizeof(d));
  fill_desc<uint32_t>(g, d);
  d.out = means;
  d.ws = ws;
  ev_kernel<6, 8, 4, uint32_t, 2, 4><<<grid, TRIOT_BLOCK, 0, (cudaStream_t)stream>>>(d);
  return cudaGetLastError() != cudaSuccess ? -100 : (int)grid;
}
