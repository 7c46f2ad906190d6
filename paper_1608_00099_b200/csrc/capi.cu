// capi.cu -- the extern "C" entry points of include/triot.h: validate (plan.cpp), pick the
// compiled instance from the dispatch tables (inst.cu), size the grid from the SM count, and
// enqueue on the caller's stream.  No device memory is allocated here.
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <mutex>
#include <utility>
#include <unordered_map>

#include "../../include/triot.h"
#include "desc.h"
#include "plan.hpp"
#include "kernels.cuh"

// dispatch tables, one per compiled family (inst.cu)
extern "C" {
const void* triot_table_0_4_0(int, int, int);
const void* triot_table_0_8_0(int, int, int);
const void* triot_table_1_4_0(int, int, int);
const void* triot_table_1_4_1(int, int, int);
const void* triot_table_1_4_2(int, int, int);
const void* triot_table_1_4_3(int, int, int);
const void* triot_table_1_8_0(int, int, int);
const void* triot_table_1_8_1(int, int, int);
const void* triot_table_1_8_2(int, int, int);
const void* triot_table_1_8_3(int, int, int);
const void* triot_table_2_4_0(int, int, int);
const void* triot_table_2_8_0(int, int, int);
const void* triot_table_2_4_1(int, int, int);
const void* triot_table_2_8_1(int, int, int);
const void* triot_table_3_4_0(int, int, int);
const void* triot_table_3_8_0(int, int, int);
const void* triot_table_4_4_0(int, int, int);
const void* triot_table_4_8_0(int, int, int);
const void* triot_table_2_4_2(int, int, int);
const void* triot_table_2_8_2(int, int, int);
const void* triot_table_5_4_0(int, int, int);
const void* triot_table_5_8_0(int, int, int);
}

namespace triot {
namespace {

typedef const void* (*TableFn)(int, int, int);

TableFn table_for(const Geom& g) {
  const bool e8 = g.esz == 8;
  if (g.op == OP_EMBED) return e8 ? triot_table_0_8_0 : triot_table_0_4_0;
  if (g.op == OP_EV && g.view) return e8 ? triot_table_2_8_2 : triot_table_2_4_2;
  if (g.op == OP_EV) return e8 ? triot_table_2_8_0 : triot_table_2_4_0;
  if (g.op == OP_DOT) return e8 ? triot_table_3_8_0 : triot_table_3_4_0;
  if (g.op == OP_UPDATE) return e8 ? triot_table_4_8_0 : triot_table_4_4_0;
  static const TableFn b4[4] = {triot_table_1_4_0, triot_table_1_4_1, triot_table_1_4_2,
                                triot_table_1_4_3};
  static const TableFn b8[4] = {triot_table_1_8_0, triot_table_1_8_1, triot_table_1_8_2,
                                triot_table_1_8_3};
  return e8 ? b8[g.binop] : b4[g.binop];
}

int vindex(const Geom& g) {
  if (g.evrows) return 5;
  if (g.dshift) return 7;
  if (g.rows) return g.rwarp ? 6 : 5;
  if (g.flat) return g.V * g.esz == 64 ? 6 : 3;  // 6: the expected value's 64-byte flat units
  if (g.V == 32 / g.esz) return 0;
  if (g.V == 16 / g.esz) return 1;
  return 2;
}

std::mutex g_mu;
int g_sms[64] = {0};
// per (device, kernel): occupancy in blocks per SM, or 1 once the kernel's dynamic shared
// memory attribute has been set on that device (attributes are per device)
struct OccKey {
  int dev;
  const void* fn;
  size_t smem = 0;  // dynamic shared memory per block the occupancy was computed for
  bool operator==(const OccKey& o) const { return dev == o.dev && fn == o.fn && smem == o.smem; }
};
struct OccHash {
  size_t operator()(const OccKey& k) const {
    return std::hash<const void*>()(k.fn) ^ ((size_t)k.dev * 0x9e3779b97f4a7c15ull) ^
           (k.smem * 0xbf58476d1ce4e5b9ull);
  }
};
std::unordered_map<OccKey, int, OccHash> g_occ;

int cuda_fail(cudaError_t e, const char* what) {
  return set_error(TRIOT_ERR_CUDA, "CUDA: %s: %s", what, cudaGetErrorString(e));
}

// The SM count of device `dev`, queried once and cached; g_mu must be held.
int sms_locked(int dev, int* sms) {
  if (dev < 0 || dev >= 64) return set_error(TRIOT_ERR_CUDA, "CUDA: device id %d", dev);
  if (!g_sms[dev]) {
    cudaError_t e = cudaDeviceGetAttribute(&g_sms[dev], cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
  }
  *sms = g_sms[dev];
  return TRIOT_OK;
}

// ---- work decomposition policy ----------------------------------
// mode 0 = each warp streams a contiguous chunk; mode 1 = grid stride (all warps sweep one
// window of the tensors together, which the B200 DRAM schedules better: tools/membench.py).
// blocks_per_sm 0 = as many as fit (occupancy).  The automatic choice was tuned on B200
// (tools/tune.py); triot_set_launch_policy() overrides it for the calling thread (tuning only).
struct Policy {
  int mode;
  int bpsm;  // > 0: blocks per SM; 0: from steps_per_warp (chunk mode) or occupancy
  int q;     // chunk mode: target steps (32-vector warp instructions) per warp
};
thread_local Policy g_override = {-1, 0, 0};

// Tuned on B200 (tools/tune.py): short contiguous chunks per warp
// (>= 4 steps of 32 vectors) in a grid of up to 64 blocks per SM -- many waves, so the hardware
// block scheduler hands out consecutive chunks as SMs free up: the active window of the tensors
// stays compact and every SM stays busy to the end.  One wave at occupancy (the first version)
// reached 5.0-5.9 TB/s on C2/C4/C5; this reaches 6.5-6.8 TB/s (single launch, clean L2).
constexpr bool kEvSplitDefault = false;
constexpr int kEvSplitBpsm = 16;
Policy auto_policy(const Geom& g) {
  if (g.op == OP_EV) return kEvSplitDefault ? Policy{0, kEvSplitBpsm, 0} : Policy{0, 0, 0};
  // inner product: one wave at occupancy, like the expected value (ncu, cold, Benchmark 2:
  // 4 blocks per SM 26.2 us vs 8 per SM 27.1 us)
  if (g.op == OP_DOT) return Policy{0, 0, 0};
  if (g.op == OP_EMBED) {
    // zero-run embeds (C5: 94 % of the steps are zero runs) keep improving up to the 4-step
    // minimum chunk (ncu, C5: 64 / 128 / 192 blocks per SM -> 160.4 / 156.6 / 156.3 us)
    Geom probe = g;
    set_decomposition(probe, 0, 1);
    if (probe.zmask) return Policy{0, 256, 0};
  }
  return Policy{0, 64, 0};
}

// One-cluster reductions (mid-size expected values): blocks per cluster, and a switch
// (TRIOT_NO_CLUSTER=1 in the environment: A/B measurements)
constexpr unsigned kClusterBlocks = 8;
std::atomic<bool> g_cluster_refused{false};  // a cluster launch failed once: the counter path from then on
bool cluster_ok() {
  static const bool off = [] { const char* e = getenv("TRIOT_NO_CLUSTER"); return e && *e == '1'; }();
  return !off && !g_cluster_refused.load(std::memory_order_relaxed);
}

int launch_geometry(const void* fn, Geom& g, int max_grid, unsigned* grid_out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  int sms, occ;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (int st = sms_locked(dev, &sms)) return st;
    auto it = g_occ.find(OccKey{dev, fn});
    if (it == g_occ.end()) {
      int nb = 0;
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, TRIOT_BLOCK, 0);
      if (e != cudaSuccess) return cuda_fail(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
      if (nb < 1) nb = 1;
      it = g_occ.emplace(OccKey{dev, fn}, nb).first;
    }
    occ = it->second;
  }
  Policy pol = auto_policy(g);
  // mode 2 (block chunks) exists only for the EV bulk-copy kernel: other kernels read the
  // descriptor per warp, so for them an override of 2 means "automatic"
  if (g_override.mode == 0 || g_override.mode == 1) pol.mode = g_override.mode;
  if (g_override.mode == 4) pol.mode = 0;
  if (g_override.bpsm > 0) pol.bpsm = g_override.bpsm;
  if ((g_override.mode == 0 || g_override.mode == 1 || g_override.mode == 4) &&
      g_override.bpsm == 0 && pol.mode != 0)
    pol.q = 0;
  const uint64_t wpb = TRIOT_BLOCK / 32;
  // >= 4 steps per warp amortise the start decode -- unless that leaves fewer than 8 blocks
  // per SM: small ops (Benchmark 3's 27 MB) are latency-bound, and more warps with one step
  // each keep more loads in flight than fewer warps with four
  uint64_t kMinSteps = g.nsteps / ((uint64_t)sms * 8 * wpb);
  if (kMinSteps > 4) kMinSteps = 4;
  if (kMinSteps < 1) kMinSteps = 1;
  uint64_t grid = (uint64_t)sms * (uint64_t)(pol.bpsm > 0 ? pol.bpsm : occ);
  if (pol.bpsm <= 0 && pol.mode == 0 && pol.q > 0)
    grid = (g.nsteps + (uint64_t)pol.q * wpb - 1) / ((uint64_t)pol.q * wpb);
  uint64_t need = (g.nsteps + kMinSteps * wpb - 1) / (kMinSteps * wpb);
  if (need < grid) grid = need;
  // a small op (less than 4 steps per warp at 8 blocks per SM) is latency-bound: keep it to one
  // wave of resident blocks (Benchmark 3's update kernel holds 2 blocks per SM at 94 registers:
  // 839 one-step blocks ran in 2.8 waves)
  if (kMinSteps < 4 && g_override.bpsm == 0 && grid > (uint64_t)sms * (uint64_t)occ)
    grid = (uint64_t)sms * (uint64_t)occ;
  if (grid > (uint64_t)max_grid) grid = (uint64_t)max_grid;
  // a reduction of at most four steps per warp of one block (32 KB: two batches of loads) runs
  // as that one block: its result needs no cross-block hand-off (ev_reduce's single-block path;
  // in a CUDA graph, per op: 128 B 2.30 -> 1.31 us, 8 KB 2.42 -> 1.56 us; tools/dbg/ev_small.py)
  if ((g.op == OP_EV || g.op == OP_DOT) && g_override.mode < 0 && g.nsteps <= 4 * wpb) grid = 1;
  // up to four steps per warp of eight blocks (256 KB): ONE thread-block cluster of 8 blocks
  // whose partials meet in block 0's shared memory (st.shared::cluster + barrier.cluster): no
  // global partial, no counter, no L2 round trips (ev_reduce's cluster path)
  g.cluster = 0;
  if ((g.op == OP_EV || g.op == OP_DOT) && g_override.mode < 0 && !g.split && grid > 1 &&
      g.nsteps <= 4 * wpb * kClusterBlocks && cluster_ok()) {
    grid = kClusterBlocks;
    g.cluster = kClusterBlocks;
  }
  if (grid < 1) grid = 1;
  set_decomposition(g, pol.mode, grid * wpb);
  if (pol.mode == 0 && !g.cluster) {  // drop blocks whose warps would get no chunk
    uint64_t q = g.wmul / 32;
    grid = (g.nsteps + q * wpb - 1) / (q * wpb);
    if (grid < 1) grid = 1;
  }
  *grid_out = (unsigned)grid;
  return TRIOT_OK;
}

// Every streaming kernel is launched with programmatic stream serialization (PDL): it may be
// scheduled while the previous kernel on the stream drains; it waits (griddepcontrol.wait)
// before its first global memory access, so results are as with plain stream order.  (B200,
// back to back in a CUDA graph: C3 5.40 vs 5.25 TB/s, C1 1.75 vs 2.03 us per op with / without;
// the latency-bound convolution is launched without it, see triot_naive_convolve.)
int launch_pdl(const void* fn, unsigned grid, unsigned block, size_t smem, cudaStream_t st,
               void** args, bool pdl = true, unsigned cluster = 0) {
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (cluster > 1) {  // the grid as thread-block clusters of `cluster` blocks (distributed smem)
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = cluster;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
  if (e != cudaSuccess) return cuda_fail(e, "cudaLaunchKernelExC");
  return TRIOT_OK;
}

template <typename IDX>
int launch_t(const Geom& g, const void* fn, unsigned grid, cudaStream_t st, void* out, void* ws) {
  Desc<IDX> d;
  memset(&d, 0, sizeof(d));
  fill_desc<IDX>(g, d);
  d.out = out;
  d.ws = ws;
  void* args[1] = {&d};
  if (g.cluster > 1) {
    // A cluster launch can be refused where 8 co-scheduled blocks do not fit (a partitioned
    // GPU): then the same grid runs the counter path -- same blocks, same fixed order -- and
    // later calls skip the cluster.
    if (launch_pdl(fn, grid, TRIOT_BLOCK, 0, st, args, true, g.cluster) == TRIOT_OK) return TRIOT_OK;
    cudaGetLastError();
    g_cluster_refused.store(true, std::memory_order_relaxed);
    d.cluster = 0;
    const int st2 = launch_pdl(fn, grid, TRIOT_BLOCK, 0, st, args);
    if (st2 == TRIOT_OK) clear_error();  // the refused attempt's message
    return st2;
  }
  return launch_pdl(fn, grid, TRIOT_BLOCK, 0, st, args);
}

// Reductions: workspace bytes a grid needs (the counter header, one P-slot partial per block).
size_t reduce_ws_bytes(uint64_t grid, int nslots) {
  return TRIOT_EV_WS_HEADER + (size_t)grid * (size_t)ev_slot_pad(nslots) * sizeof(double);
}

// EV bulk-copy fast path: full 32-byte vectors, 32-B aligned p, one persistent block per SM
int launch_ev_tma(Geom& g, void* stream, void* out, void* ws, size_t ws_bytes, bool* used) {
  *used = false;
  if (g.op != OP_EV || g.view || g.flat || g.V * g.esz != 32 || !g.t[0].vec) return TRIOT_OK;
  // measured on B200 (ncu, cold cache, C3): the lean 32-B-load kernel at one full wave of 4
  // blocks/SM takes 30.2 us, the bulk-copy pipeline 33.1 us -> the bulk-copy path is opt-in
  if (g_override.mode != 2 && g_override.mode != 3) return TRIOT_OK;
  // mode 2: one persistent 512-thread block per SM, 6 x 32 KB stages; mode 3: small stages
  // (4 x 16 KB, 256 threads, several blocks per SM, many blocks)
  const bool small = g_override.mode == 3;
  const int block = small ? TRIOT_EVS_BLOCK : TRIOT_EV_TMA_BLOCK;
  const int smem = small ? TRIOT_EVS_SMEM : TRIOT_EV_SMEM;
  const void* fn =
      (g.esz == 8 ? triot_table_2_8_1 : triot_table_2_4_1)(g.D, small ? 1 : 0, g.idx64 ? 1 : 0);
  if (!fn) return TRIOT_OK;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  int sms;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (int st = sms_locked(dev, &sms)) return st;
    if (g_occ.find(OccKey{dev, fn}) == g_occ.end()) {
      e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
      g_occ.emplace(OccKey{dev, fn}, 1);
    }
  }
  uint64_t blocks = (uint64_t)sms * (uint64_t)(g_override.bpsm > 0 ? g_override.bpsm : 1);
  const uint64_t svec = small ? TRIOT_EVS_SVEC : TRIOT_EV_SVEC;
  uint64_t need = (g.nvec + svec - 1) / svec;
  if (need < blocks) blocks = need;
  if (blocks > TRIOT_EV_MAX_GRID) blocks = TRIOT_EV_MAX_GRID;
  if (blocks < 1) blocks = 1;
  set_decomposition(g, 2, blocks);
  g.dv = (uint64_t)block;  // threads step by one block
  set_step(g);
  uint64_t grid = (g.nvec + g.wmul - 1) / g.wmul;
  size_t need_ws = reduce_ws_bytes(grid, g.D + 2);
  if (!ws || ws_bytes < need_ws)
    return set_error(TRIOT_ERR_WORKSPACE, "Workspace: %zu bytes given, %zu needed", ws_bytes,
                     need_ws);
  *used = true;
  auto go = [&](auto tag) -> int {
    using IDX = decltype(tag);
    Desc<IDX> d;
    memset(&d, 0, sizeof(d));
    fill_desc<IDX>(g, d);
    d.out = out;
    d.ws = ws;
    void* args[1] = {&d};
    return launch_pdl(fn, (unsigned)grid, block, smem, (cudaStream_t)stream, args);
  };
  return g.idx64 ? go(uint64_t(0)) : go(uint32_t(0));
}

// Dense EV with a short odd innermost extent (plan_ev_rows): tiles of whole rows staged in
// shared memory by bulk copies, one wave of blocks at occupancy, contiguous tiles per block.
int launch_ev_rows(Geom& g, void* stream, void* out, void* ws, size_t ws_bytes) {
  const void* fn = table_for(g)(g.D, 5, g.idx64 ? 1 : 0);
  if (!fn) return set_error(TRIOT_ERR_CUDA, "internal: no EV row-tile instance for D=%d", g.D);
  const uint64_t rb = (uint64_t)g.rowlen * (uint64_t)g.esz;
  uint64_t rpt = TRIOT_EVROWS_STAGE / ((uint64_t)TRIOT_BLOCK * rb);  // ~16 KB stages
  if (rpt < 1) rpt = 1;
  if (rpt > 8) rpt = 8;
  // Tiny odd rows (at most 32 bytes): a thread takes rpt CONSECUTIVE rows of a tile, so that
  // between them the digits advance by Alg 3's +1 (one subtraction in the common case) instead
  // of a full mixed-radix step per 12-28 bytes; rpt odd keeps the threads' shared-memory
  // strides (rpt * n words) odd, i.e. conflict-free.  TRIOT_EVROWS_NOGROUP=1: off (A/B).
  static const bool nogroup = [] { const char* e = getenv("TRIOT_EVROWS_NOGROUP"); return e && *e == '1'; }();
  const bool grouped = !nogroup && rb <= 32 && (g.rowlen & 1u) && rpt >= 3;
  if (grouped && (rpt & 1) == 0) --rpt;
  const uint64_t stage = ((uint64_t)TRIOT_BLOCK * rpt * rb + 127) & ~127ull;
  const size_t smem = (size_t)(kEvRowsStages * stage + 8 * kEvRowsStages);
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  int sms, occ = 1;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (int st = sms_locked(dev, &sms)) return st;
    // the attribute is the largest stage set any row length can ask for (n <= 31, f64: one
    // row per thread, 3 x 63.5 KB), set once per device; the occupancy per stage size
    if (g_occ.find(OccKey{dev, fn, 1}) == g_occ.end()) {
      const int maxsmem = kEvRowsStages * TRIOT_BLOCK * 31 * 8 + 8 * kEvRowsStages + 128;
      e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsmem);
      if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
      g_occ.emplace(OccKey{dev, fn, 1}, 1);
    }
    auto it = g_occ.find(OccKey{dev, fn, smem});
    if (it == g_occ.end()) {
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, TRIOT_BLOCK, smem);
      if (e != cudaSuccess) return cuda_fail(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
      if (occ < 1) occ = 1;
      it = g_occ.emplace(OccKey{dev, fn, smem}, occ).first;
    }
    occ = it->second;
  }
  const uint64_t tr = (uint64_t)TRIOT_BLOCK * rpt;
  const uint64_t ntiles = (g.nvec + tr - 1) / tr;
  uint64_t blocks = (uint64_t)sms * (uint64_t)(g_override.bpsm > 0 ? g_override.bpsm : occ);
  if (blocks > TRIOT_EV_MAX_GRID) blocks = TRIOT_EV_MAX_GRID;
  if (blocks > ntiles) blocks = ntiles;
  if (blocks < 1) blocks = 1;
  const uint64_t per = (ntiles + blocks - 1) / blocks;
  const uint64_t grid = (ntiles + per - 1) / per;
  g.mode = 0;
  // a thread's rows advance by one block's worth; grouped: from the last row of its group to
  // the first row of its group in the next tile
  g.dv = grouped ? tr - rpt + 1 : (uint64_t)TRIOT_BLOCK;
  set_step(g);
  g.wmul = tr;
  g.wspan = per;
  g.rwin = (uint32_t)rpt;
  g.rmag = (uint32_t)stage;
  const size_t need = reduce_ws_bytes(grid, g.D + 2);
  if (!ws || ws_bytes < need)
    return set_error(TRIOT_ERR_WORKSPACE, "Workspace: %zu bytes given, %zu needed", ws_bytes, need);
  auto go = [&](auto tag) -> int {
    using IDX = decltype(tag);
    Desc<IDX> d;
    memset(&d, 0, sizeof(d));
    fill_desc<IDX>(g, d);
    d.out = out;
    d.ws = ws;
    d.rgroup = grouped ? 1u : 0u;
    void* args[1] = {&d};
    return launch_pdl(fn, (unsigned)grid, TRIOT_BLOCK, smem, (cudaStream_t)stream, args);
  };
  return g.idx64 ? go(uint64_t(0)) : go(uint32_t(0));
}

// ---- EV of a view window with rows of 32..256 elements: TMA tensor tiles (ev_view_tma_kernel)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  });
  return fn;
}

// Returns TRIOT_OK with *used = false when the view does not qualify (the regular view kernel
// then runs): rank of the window's non-unit axes 2..5, its innermost axis the base's innermost
// with 32..256 elements, a 16-byte aligned base whose row pitch and outer strides are multiples
// of 16 bytes.
int launch_ev_view_tma(const Geom& g, const triot_view* v, int d, int dtype, bool with_mass,
                       void* out, void* ws, size_t ws_bytes, void* stream, bool* used) {
  *used = false;
  if (g_override.mode >= 0 || !rows_enabled()) return TRIOT_OK;  // tuning runs keep the old path
  const int esz = dtype == TRIOT_F32 ? 4 : 8;
  int ax[TRIOT_MAXD], m = 0;
  for (int k = 0; k < d; ++k)
    if (v->shape[k] > 1) ax[m++] = k;
  if (m < 2 || m > 5 || ax[m - 1] != d - 1) return TRIOT_OK;
  const uint64_t n = (uint64_t)v->shape[d - 1];
  if (n < 32 || n > 256) return TRIOT_OK;
  if (((uintptr_t)v->data) % 16) return TRIOT_OK;
  uint64_t bstride[TRIOT_MAXD];  // base strides in bytes
  uint64_t acc = (uint64_t)esz;
  for (int k = d - 1; k >= 0; --k) {
    bstride[k] = acc;
    acc *= (uint64_t)v->base_shape[k];
  }
  for (int j = 0; j < m - 1; ++j)
    if (bstride[ax[j]] % 16 || bstride[ax[j]] >= (1ull << 40)) return TRIOT_OK;
  for (int j = 0; j < m; ++j)  // TMA coordinates are 32-bit signed
    if (v->base_shape[ax[j]] >= (1ll << 31)) return TRIOT_OK;
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return TRIOT_OK;
  // the unit axes of the window fold into the map's base address (multiples of 16 bytes)
  uint64_t bias = 0;
  for (int k = 0; k < d; ++k)
    if (v->shape[k] == 1 && v->start) bias += (uint64_t)v->start[k] * bstride[k];
  // the box starts on a 16-byte boundary at or before the window's first column
  const uint64_t s_in = v->start ? (uint64_t)v->start[d - 1] : 0;
  const uint32_t cshift = (uint32_t)((s_in * esz % 16) / esz);
  const uint32_t nbox = (uint32_t)(((n + cshift) * esz + 15) / 16 * 16 / esz);
  if (nbox > 256) return TRIOT_OK;
  const int D = m - 1;
  EvTmaGeo G;
  memset(&G, 0, sizeof(G));
  G.m = (uint32_t)m;
  G.n = (uint32_t)n;
  G.nbox = nbox;
  G.cshift = cshift;
  cuuint64_t gdim[5], gstr[4];
  cuuint32_t box[5], estr[5];
  for (int j = 0; j < m; ++j) {  // TMA dim j = window axis ax[m-1-j]
    const int k = ax[m - 1 - j];
    gdim[j] = (cuuint64_t)v->base_shape[k];
    if (j) gstr[j - 1] = (cuuint64_t)bstride[k];
    G.coord0[j] = (int32_t)(v->start ? v->start[k] : 0) - (j == 0 ? (int32_t)cshift : 0);
    box[j] = 1;
    estr[j] = 1;
  }
  for (int j = 0; j < D; ++j) G.ext[j] = (uint64_t)v->shape[ax[j]];
  uint64_t R = 16384 / ((uint64_t)nbox * esz);
  if (R < 1) R = 1;
  if (R > 256) R = 256;
  if (R > G.ext[D - 1]) R = G.ext[D - 1];
  box[0] = nbox;
  box[1] = (cuuint32_t)R;
  G.R = (uint32_t)R;
  G.stage = (uint32_t)(((uint64_t)nbox * R * esz + 127) & ~127ull);
  G.tpa = (G.ext[D - 1] + R - 1) / R;
  G.ntiles = G.tpa;
  for (int j = 0; j < D - 1; ++j) G.ntiles *= G.ext[j];
  if (G.ntiles >= (1ull << 32) || G.ext[D - 1] >= (1ull << 31)) return TRIOT_OK;  // 32-bit tiles
  CUtensorMap map;
  CUresult cr = enc(&map, esz == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                    (cuuint32_t)m, (char*)v->data + bias, gdim, gstr, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return TRIOT_OK;  // not encodable: the regular kernel
  const void* fns4[4] = {(const void*)&ev_view_tma_kernel<1, 4>, (const void*)&ev_view_tma_kernel<2, 4>,
                         (const void*)&ev_view_tma_kernel<3, 4>, (const void*)&ev_view_tma_kernel<4, 4>};
  const void* fns8[4] = {(const void*)&ev_view_tma_kernel<1, 8>, (const void*)&ev_view_tma_kernel<2, 8>,
                         (const void*)&ev_view_tma_kernel<3, 8>, (const void*)&ev_view_tma_kernel<4, 8>};
  const void* fn = (esz == 4 ? fns4 : fns8)[D - 1];
  const size_t smem = (size_t)kEvRowsStages * G.stage + 8 * kEvRowsStages;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  int sms, occ = 1;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (int st = sms_locked(dev, &sms)) return st;
    if (g_occ.find(OccKey{dev, fn, 1}) == g_occ.end()) {
      e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               kEvRowsStages * 20480 + 8 * kEvRowsStages);
      if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
      g_occ.emplace(OccKey{dev, fn, 1}, 1);
    }
    auto it = g_occ.find(OccKey{dev, fn, smem});
    if (it == g_occ.end()) {
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, TRIOT_BLOCK, smem);
      if (e != cudaSuccess) return cuda_fail(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
      if (occ < 1) occ = 1;
      it = g_occ.emplace(OccKey{dev, fn, smem}, occ).first;
    }
    occ = it->second;
  }
  uint64_t blocks = (uint64_t)sms * (uint64_t)occ;
  if (blocks > TRIOT_EV_MAX_GRID) blocks = TRIOT_EV_MAX_GRID;
  if (blocks > G.ntiles) blocks = G.ntiles;
  if (blocks < 1) blocks = 1;
  G.per = (G.ntiles + blocks - 1) / blocks;
  const uint64_t grid = (G.ntiles + G.per - 1) / G.per;
  const size_t need = reduce_ws_bytes(grid, D + 2);
  if (!ws || ws_bytes < need)
    return set_error(TRIOT_ERR_WORKSPACE, "Workspace: %zu bytes given, %zu needed", ws_bytes, need);
  Desc<uint32_t> desc;
  memset(&desc, 0, sizeof(desc));
  desc.out = out;
  desc.ws = ws;
  desc.d_out = d + (with_mass ? 1 : 0);
  for (int k = 0; k <= TRIOT_MAXD; ++k) desc.slot_of_axis[k] = -1;
  for (int j = 0; j < m; ++j) desc.slot_of_axis[ax[j]] = j;  // outer digits j < D; inner D
  desc.slot_of_axis[d] = D + 1;                              // the mass
  void* args[3] = {&desc, &map, &G};
  *used = true;
  (void)g;
  return launch_pdl(fn, (unsigned)grid, TRIOT_BLOCK, smem, (cudaStream_t)stream, args);
}

int launch(Geom& g, void* stream, void* out, void* ws, size_t ws_bytes) {
  if (g.op == OP_EV && g.evrows) return launch_ev_rows(g, stream, out, ws, ws_bytes);
  if (g.op == OP_EV) {
    bool used = false;
    int st = launch_ev_tma(g, stream, out, ws, ws_bytes, &used);
    if (st || used) return st;
  }
  const void* fn = table_for(g)(g.D, vindex(g), g.idx64 ? 1 : 0);
  if (!fn) return set_error(TRIOT_ERR_CUDA, "internal: no instance for D=%d V=%d", g.D, g.V);
  const bool red = g.op == OP_EV || g.op == OP_DOT;
  // EV: partials per block summed by ev_final_kernel (PDL) instead of the last block (mode 4)
  g.split = g.op == OP_EV && (g_override.mode == 4 || (g_override.mode < 0 && kEvSplitDefault));
  int max_grid = 1 << 30;
  if (red) max_grid = TRIOT_EV_MAX_GRID;
  unsigned grid;
  int st = launch_geometry(fn, g, max_grid, &grid);
  if (st) return st;
  if (g.zmask) {  // embed with zero runs (set_step): its own instance, same geometry
    fn = table_for(g)(g.D, 4, g.idx64 ? 1 : 0);
    if (!fn) return set_error(TRIOT_ERR_CUDA, "internal: no zero-run instance for D=%d", g.D);
  }
  if (g.op == OP_EV || g.op == OP_DOT) {
    size_t need = reduce_ws_bytes(grid, g.op == OP_DOT ? 1 : g.D + 2);
    if (!ws || ws_bytes < need)
      return set_error(TRIOT_ERR_WORKSPACE, "Workspace: %zu bytes given, %zu needed", ws_bytes,
                       need);
  }
  cudaStream_t s = (cudaStream_t)stream;
  int st2 = g.idx64 ? launch_t<uint64_t>(g, fn, grid, s, out, ws)
                    : launch_t<uint32_t>(g, fn, grid, s, out, ws);
  if (st2 || !g.split) return st2;
  EvFin f;
  memset(&f, 0, sizeof(f));
  f.part = (const double*)((const char*)ws + TRIOT_EV_WS_HEADER);
  f.out = (double*)out;
  f.nblk = grid;
  f.ns = g.D + 2;
  f.d_out = g.nout >= 0 ? g.nout : g.d + (g.with_mass ? 1 : 0);
  for (int k = 0; k <= TRIOT_MAXD; ++k) f.slot_of_axis[k] = g.slot_of_axis[k];
  f.nax = g.nax;
  for (int k = 0; k < TRIOT_MAXD; ++k) f.offd[k] = g.offd[k];
  void* args[1] = {&f};
  return launch_pdl((const void*)&ev_final_kernel<kFinBlock>, 1, kFinBlock, 0, s, args);
}

size_t ev_ws_bytes(int nslots) { return reduce_ws_bytes(TRIOT_EV_MAX_GRID, nslots); }

// ---- plan cache (dense embed / apply_binary): repeated calls on the same shapes skip the
// planner and the launch geometry (P:266 calls the dispatch "already a prerequisite cost"; on a
// 75 KB op it is most of the host time).  The plan depends on the pointers only through their
// alignment (modulo 32) and null-ness -- both in the key -- and through the aliasing checks,
// which are re-run on every hit: any overlap between the tensors (allowed in-place binary calls
// included) takes the full planner, so every error is reported exactly as without the cache.
struct PlanKey {
  int32_t op, d, dtype, sub, dev, pmode, pbpsm, rows_on;
  int64_t sh[4][TRIOT_MAXD];  // tensor shapes (+ the iteration shape for binary)
  uint8_t has[4], mod[3];
  bool operator==(const PlanKey& o) const { return memcmp(this, &o, sizeof(PlanKey)) == 0; }
};
struct PlanEntry {
  PlanKey key;
  bool valid = false;
  Geom g;
  const void* fn = nullptr;
  unsigned grid = 0;
};
constexpr int kPlanCache = 8;
thread_local PlanEntry g_plans[kPlanCache];

uint64_t key_hash(const PlanKey& k) {
  const unsigned char* b = (const unsigned char*)&k;
  uint64_t h = 1469598103934665603ull;
  for (size_t i = 0; i < sizeof(PlanKey); ++i) h = (h ^ b[i]) * 1099511628211ull;
  return h;
}

bool make_key(PlanKey& k, int op, int d, int dtype, int sub, const void* const* ptrs,
              const int64_t* const* shapes, int nt, const int64_t* iter) {
  if (d < 1 || d > TRIOT_MAXD) return false;
  memset(&k, 0, sizeof(k));
  k.op = op;
  k.d = d;
  k.dtype = dtype;
  k.sub = sub;
  if (cudaGetDevice(&k.dev) != cudaSuccess) return false;
  k.pmode = g_override.mode;
  k.pbpsm = g_override.bpsm;
  k.rows_on = rows_enabled() ? 1 : 0;
  for (int x = 0; x < nt; ++x) {
    k.has[x] = shapes[x] ? 1 : 0;
    if (shapes[x]) memcpy(k.sh[x], shapes[x], sizeof(int64_t) * d);
    k.mod[x] = (uint8_t)(((uintptr_t)ptrs[x] & 31u) | (ptrs[x] ? 0x80u : 0u));
  }
  k.has[3] = iter ? 1 : 0;
  if (iter) memcpy(k.sh[3], iter, sizeof(int64_t) * d);
  return true;
}

// A hit with no overlap among the tensors: the cached plan with this call's pointers.
bool plan_hit(const PlanKey& k, const void* const* ptrs, int nt, Geom& g, const void** fn,
              unsigned* grid) {
  PlanEntry& e = g_plans[key_hash(k) % kPlanCache];
  if (!e.valid || !(e.key == k)) return false;
  for (int x = 0; x < nt; ++x)
    for (int y = x + 1; y < nt; ++y)
      if (ptrs[x] && ptrs[y]) {
        const uintptr_t a0 = (uintptr_t)ptrs[x], a1 = a0 + e.g.t[x].numel * (uint64_t)e.g.esz;
        const uintptr_t b0 = (uintptr_t)ptrs[y], b1 = b0 + e.g.t[y].numel * (uint64_t)e.g.esz;
        if (e.g.t[x].numel && e.g.t[y].numel && a0 < b1 && b0 < a1) return false;
      }
  g = e.g;
  for (int x = 0; x < nt; ++x) g.t[x].ptr = ptrs[x];
  *fn = e.fn;
  *grid = e.grid;
  return true;
}

void plan_store(const PlanKey& k, const Geom& g, const void* fn, unsigned grid) {
  PlanEntry& e = g_plans[key_hash(k) % kPlanCache];
  e.key = k;
  e.g = g;
  e.fn = fn;
  e.grid = grid;
  e.valid = true;
}

// embed / binary: choose the instance and the grid (the part of launch() a plan-cache hit skips)
int prepare_stream_op(Geom& g, const void** fn_out, unsigned* grid_out) {
  const void* fn = table_for(g)(g.D, vindex(g), g.idx64 ? 1 : 0);
  if (!fn) return set_error(TRIOT_ERR_CUDA, "internal: no instance for D=%d V=%d", g.D, g.V);
  unsigned grid;
  int st = launch_geometry(fn, g, 1 << 30, &grid);
  if (st) return st;
  if (g.zmask) {  // embed with zero runs (set_step): its own instance, same geometry
    fn = table_for(g)(g.D, 4, g.idx64 ? 1 : 0);
    if (!fn) return set_error(TRIOT_ERR_CUDA, "internal: no zero-run instance for D=%d", g.D);
  }
  *fn_out = fn;
  *grid_out = grid;
  return TRIOT_OK;
}

int launch_stream_op(const Geom& g, const void* fn, unsigned grid, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  return g.idx64 ? launch_t<uint64_t>(g, fn, grid, s, nullptr, nullptr)
                 : launch_t<uint32_t>(g, fn, grid, s, nullptr, nullptr);
}

}  // namespace
}  // namespace triot

using namespace triot;

extern "C" {

int triot_max_dimension(void) { return TRIOT_MAXD; }

const char* triot_status_string(int s) {
  switch (s) {
    case TRIOT_OK: return "TRIOT_OK";
    case TRIOT_ERR_NULL_POINTER: return "TRIOT_ERR_NULL_POINTER";
    case TRIOT_ERR_UNSUPPORTED_DIMENSION: return "TRIOT_ERR_UNSUPPORTED_DIMENSION";
    case TRIOT_ERR_BAD_SHAPE: return "TRIOT_ERR_BAD_SHAPE";
    case TRIOT_ERR_AXIS_OUT_OF_BOUNDS: return "TRIOT_ERR_AXIS_OUT_OF_BOUNDS";
    case TRIOT_ERR_BAD_DTYPE_OR_OP: return "TRIOT_ERR_BAD_DTYPE_OR_OP";
    case TRIOT_ERR_MISALIGNED: return "TRIOT_ERR_MISALIGNED";
    case TRIOT_ERR_ALIASING: return "TRIOT_ERR_ALIASING";
    case TRIOT_ERR_WORKSPACE: return "TRIOT_ERR_WORKSPACE";
    case TRIOT_ERR_CUDA: return "TRIOT_ERR_CUDA";
    default: return "TRIOT_ERR_UNKNOWN";
  }
}

const char* triot_last_error(void) { return last_error(); }

int triot_embed(void* dst, const int64_t* dst_shape, const void* src, const int64_t* src_shape,
                int d, int dtype, unsigned flags, void* cuda_stream) {
  const void* ptrs[2] = {dst, src};
  const int64_t* shapes[2] = {dst_shape, src_shape};
  PlanKey key;
  const bool keyed = dst_shape && src_shape && make_key(key, OP_EMBED, d, dtype, (int)flags, ptrs,
                                                        shapes, 2, nullptr);
  Geom g;
  const void* fn;
  unsigned grid;
  if (keyed && plan_hit(key, ptrs, 2, g, &fn, &grid)) {
    const int st0 = launch_stream_op(g, fn, grid, cuda_stream);
    if (!st0) clear_error();
    return st0;
  }
  int st = plan_embed(g, dst, dst_shape, src, src_shape, d, dtype, flags);
  if (st || g.empty) return st;
  if ((st = prepare_stream_op(g, &fn, &grid))) return st;
  if (keyed) plan_store(key, g, fn, grid);
  st = launch_stream_op(g, fn, grid, cuda_stream);
  if (!st) clear_error();
  return st;
}

int triot_apply_binary(void* c, const int64_t* c_shape, const void* a, const int64_t* a_shape,
                       const void* b, const int64_t* b_shape, const int64_t* iter_shape, int d,
                       int dtype, int op, void* cuda_stream) {
  const void* ptrs[3] = {c, a, b};
  const int64_t* shapes[3] = {c_shape, a_shape, b_shape};
  PlanKey key;
  const bool keyed = a_shape && b_shape &&
                     make_key(key, OP_BINARY, d, dtype, op, ptrs, shapes, 3, iter_shape);
  Geom g;
  const void* fn;
  unsigned grid;
  if (keyed && plan_hit(key, ptrs, 3, g, &fn, &grid)) {
    const int st0 = launch_stream_op(g, fn, grid, cuda_stream);
    if (!st0) clear_error();
    return st0;
  }
  int st = plan_binary(g, c, c_shape, a, a_shape, b, b_shape, iter_shape, d, dtype, op);
  if (st || g.empty) return st;
  if ((st = prepare_stream_op(g, &fn, &grid))) return st;
  if (keyed) plan_store(key, g, fn, grid);
  st = launch_stream_op(g, fn, grid, cuda_stream);
  if (!st) clear_error();
  return st;
}

int triot_embed_view(const triot_view* dst, const triot_view* src, int d, int dtype,
                     unsigned flags, void* cuda_stream) {
  Geom g;
  int st = plan_embed_view(g, dst, src, d, dtype, flags);
  if (st || g.empty) return st;
  st = launch(g, cuda_stream, nullptr, nullptr, 0);
  if (!st) clear_error();
  return st;
}

int triot_apply_binary_view(const triot_view* c, const triot_view* a, const triot_view* b,
                            const int64_t* iter_shape, int d, int dtype, int op,
                            void* cuda_stream) {
  Geom g;
  int st = plan_binary_view(g, c, a, b, iter_shape, d, dtype, op);
  if (st || g.empty) return st;
  st = launch(g, cuda_stream, nullptr, nullptr, 0);
  if (!st) clear_error();
  return st;
}

int triot_inner_product_workspace_size(size_t* bytes) {
  if (!bytes) return set_error(TRIOT_ERR_NULL_POINTER, "NullPointer: bytes is NULL");
  *bytes = ev_ws_bytes(1);
  return TRIOT_OK;
}

int triot_inner_product(double* out, const void* a, const int64_t* a_shape, const void* b,
                        const int64_t* b_shape, const int64_t* iter_shape, int d, int dtype,
                        void* workspace, size_t workspace_bytes, void* cuda_stream) {
  Geom g;
  int st = plan_dot(g, a, a_shape, b, b_shape, iter_shape, d, dtype);
  if (st) return st;
  if (!out) return set_error(TRIOT_ERR_NULL_POINTER, "NullPointer: out is NULL");
  if (((uintptr_t)out) % 8)
    return set_error(TRIOT_ERR_MISALIGNED, "Misaligned: out is not 8-byte aligned");
  if (g.empty) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double), (cudaStream_t)cuda_stream);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
    clear_error();
    return TRIOT_OK;
  }
  st = launch(g, cuda_stream, out, workspace, workspace_bytes);
  if (!st) clear_error();
  return st;
}

int triot_fused_update(void* x, const int64_t* x_shape, const void* y, const int64_t* y_shape,
                       const void* z, const int64_t* z_shape, int d, int dtype,
                       void* cuda_stream) {
  Geom g;
  int st = plan_update(g, x, x_shape, y, y_shape, z, z_shape, d, dtype);
  if (st || g.empty) return st;
  st = launch(g, cuda_stream, nullptr, nullptr, 0);
  if (!st) clear_error();
  return st;
}

int triot_naive_convolve(void* result, const void* lhs, const int64_t* lhs_shape,
                         const void* rhs, const int64_t* rhs_shape, int d, int dtype,
                         void* cuda_stream) {
  Geom g;
  int st = plan_conv(g, result, lhs, lhs_shape, rhs, rhs_shape, d, dtype);
  if (st) return st;
  // Few outputs (the paper's Benchmark 4: 7,665) cannot fill the SMs one lane per output, so G
  // lanes share an output (group kernel: latency-bound on the add chain, 28 us); with >= 8 warps
  // of outputs per SM the lane-per-output kernel issues ~6x fewer instructions per term.  It
  // iterates the smaller operand's index space (reversed order when that is rhs: tensors 0/1
  // and their extents swap).  Policy mode 1 forces the group kernel, mode 0 the lane kernel.
  int sms = 148;  // the B200's count if the query fails (only the kernel choice depends on it)
  {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) {
      std::lock_guard<std::mutex> lk(g_mu);
      int q = 0;
      if (sms_locked(dev, &q) == TRIOT_OK) sms = q;
    }
  }
  const bool group = g_override.mode == 1 ||
                     (g_override.mode != 0 && g.nvec < (uint64_t)sms * 8 * 32);
  const bool rev = !group && g.t[1].numel < g.t[0].numel;
  if (rev) {
    std::swap(g.t[0], g.t[1]);
    for (int k = 0; k < g.D; ++k) std::swap(g.bnd[k], g.dlt[k]);
  }
  // stage both operands in shared memory when they fit (<= 96 KB together)
  const uint64_t nl_pad = (g.t[0].numel + 3) & ~3ull;
  const size_t smem = (size_t)(nl_pad + g.t[1].numel) * (size_t)g.esz;
  const bool use_smem = smem <= 96 * 1024;
  const void* fn = (g.esz == 8 ? triot_table_5_8_0 : triot_table_5_4_0)(
      g.D, group ? 2 : (rev ? 1 : 0), use_smem ? 1 : 0);
  if (!fn) return set_error(TRIOT_ERR_CUDA, "internal: no convolution instance for d=%d", d);
  if (use_smem) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_occ.find(OccKey{dev, fn}) == g_occ.end()) {
      e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
      if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
      g_occ.emplace(OccKey{dev, fn}, 1);
    }
  }
  Desc<uint32_t> desc;
  memset(&desc, 0, sizeof(desc));
  fill_desc<uint32_t>(g, desc);
  desc.out = result;
  desc.t[0].rho = (uint32_t)g.t[0].numel;  // operand element counts for the staging loop
  desc.t[1].rho = (uint32_t)g.t[1].numel;
  desc.t[0].numel_pad = (uint32_t)nl_pad;
  void* args[1] = {&desc};
  const unsigned block = group ? TRIOT_CONV_BLOCK : kConvLaneBlock;
  const uint64_t per_block = group ? TRIOT_CONV_BLOCK / TRIOT_CONV_GROUP : kConvLaneBlock;
  unsigned grid = (unsigned)((g.nvec + per_block - 1) / per_block);
  // Plain stream order, not PDL: a successor's blocks made resident early by the programmatic
  // launch slow this latency-bound kernel down (B200, 50 Benchmark-4 calls in a CUDA graph:
  // 43.3 us per call with PDL, 24.0 us without); its griddepcontrol instructions are no-ops then.
  st = launch_pdl(fn, grid, block, use_smem ? smem : 0, (cudaStream_t)cuda_stream, args,
                  /*pdl=*/false);
  if (!st) clear_error();
  return st;
}

int triot_expected_value_workspace_size(const int64_t* shape, int d, int dtype, size_t* bytes) {
  if (!bytes) return set_error(TRIOT_ERR_NULL_POINTER, "NullPointer: bytes is NULL");
  Geom g;
  // validate the shape exactly like the real call (pointer checks skipped: no data yet)
  int st = plan_ev(g, (const void*)(uintptr_t)64, shape, d, dtype);
  if (st) return st;
  *bytes = ev_ws_bytes(d + 2);
  return TRIOT_OK;
}

static int expected_value_impl(double* means, const void* p, const int64_t* shape, int d,
                               int dtype, void* workspace, size_t workspace_bytes,
                               void* cuda_stream, bool with_mass,
                               const triot_view* pv = nullptr, const int64_t* offset = nullptr) {
  Geom g;
  int st = pv ? plan_ev_view(g, pv, d, dtype) : plan_ev(g, p, shape, d, dtype);
  if (st) return st;
  if (pv) p = g.t[0].ptr;
  g.with_mass = with_mass;
  if (offset) {  // the coordinates of p's element 0 in a larger PMF (P:607 slabs)
    for (int k = 0; k < d; ++k) {
      if (offset[k] < 0 || offset[k] > (int64_t)(1ll << 53))
        return set_error(TRIOT_ERR_BAD_SHAPE, "BadShape: offset[%d] = %lld outside [0, 2^53]", k,
                         (long long)offset[k]);
      g.offd[k] = (double)offset[k];
    }
    g.nax = d;
  }
  const int nout = d + (with_mass ? 1 : 0);
  if (!means) return set_error(TRIOT_ERR_NULL_POINTER, "NullPointer: means is NULL");
  if (((uintptr_t)means) % 8)
    return set_error(TRIOT_ERR_MISALIGNED, "Misaligned: means is not 8-byte aligned");
  {
    uintptr_t m0 = (uintptr_t)means, m1 = m0 + (uintptr_t)nout * 8;
    uintptr_t p0 = (uintptr_t)p, p1 = p0 + (uintptr_t)g.t[0].numel * (uintptr_t)g.esz;
    if (pv) {  // the view's whole base buffer
      uint64_t nb = 1;
      for (int k = 0; k < d; ++k) nb *= (uint64_t)pv->base_shape[k];
      p0 = (uintptr_t)pv->data;
      p1 = p0 + (uintptr_t)nb * (uintptr_t)g.esz;
    }
    if (g.t[0].numel && m0 < p1 && p0 < m1)
      return set_error(TRIOT_ERR_ALIASING, "Aliasing: means overlaps p");
  }
  if (pv && !g.empty && !offset) {  // long view rows: TMA tensor tiles
    bool used = false;
    st = launch_ev_view_tma(g, pv, d, dtype, with_mass, means, workspace, workspace_bytes,
                            cuda_stream, &used);
    if (st || used) {
      if (!st) clear_error();
      return st;
    }
  }
  if (g.empty) {  // empty sums: 0 (the offsets multiply a zero mass)
    cudaError_t e =
        cudaMemsetAsync(means, 0, (size_t)nout * sizeof(double), (cudaStream_t)cuda_stream);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
    clear_error();
    return TRIOT_OK;
  }
  st = launch(g, cuda_stream, means, workspace, workspace_bytes);
  if (!st) clear_error();
  return st;
}

int triot_expected_value(double* means, const void* p, const int64_t* shape, int d, int dtype,
                         void* workspace, size_t workspace_bytes, void* cuda_stream) {
  return expected_value_impl(means, p, shape, d, dtype, workspace, workspace_bytes, cuda_stream,
                             false);
}

int triot_expected_value_mass(double* out, const void* p, const int64_t* shape, int d, int dtype,
                              void* workspace, size_t workspace_bytes, void* cuda_stream) {
  return expected_value_impl(out, p, shape, d, dtype, workspace, workspace_bytes, cuda_stream,
                             true);
}

int triot_expected_value_offset(double* out, const void* p, const int64_t* shape,
                                const int64_t* offset, int d, int dtype, int with_mass,
                                void* workspace, size_t workspace_bytes, void* cuda_stream) {
  return expected_value_impl(out, p, shape, d, dtype, workspace, workspace_bytes, cuda_stream,
                             with_mass != 0, nullptr, offset);
}

int triot_sum_rows(double* out, const double* rows, int64_t nrows, int64_t ncols,
                   void* cuda_stream) {
  if (ncols < 0 || nrows < 0)
    return set_error(TRIOT_ERR_BAD_SHAPE, "BadShape: nrows %lld, ncols %lld", (long long)nrows,
                     (long long)ncols);
  if (ncols == 0) return TRIOT_OK;
  if (!out || (nrows && !rows)) return set_error(TRIOT_ERR_NULL_POINTER, "NullPointer: out/rows");
  if (((uintptr_t)out) % 8 || ((uintptr_t)rows) % 8)
    return set_error(TRIOT_ERR_MISALIGNED, "Misaligned: out/rows not 8-byte aligned");
  {
    uintptr_t o0 = (uintptr_t)out, o1 = o0 + (uintptr_t)ncols * 8;
    uintptr_t r0 = (uintptr_t)rows, r1 = r0 + (uintptr_t)(nrows * ncols) * 8;
    if (nrows && o0 < r1 && r0 < o1) return set_error(TRIOT_ERR_ALIASING, "Aliasing: out overlaps rows");
  }
  const unsigned grid = (unsigned)((ncols + 255) / 256);
  const double* r = rows;
  double* o = out;
  uint64_t nr = (uint64_t)nrows, nc = (uint64_t)ncols;
  void* args[4] = {&o, &r, &nr, &nc};
  int st = launch_pdl((const void*)&sum_rows_kernel<256>, grid, 256, 0, (cudaStream_t)cuda_stream,
                      args);
  if (!st) clear_error();
  return st;
}

int triot_expected_value_view(double* out, const triot_view* p, int d, int dtype, int with_mass,
                              void* workspace, size_t workspace_bytes, void* cuda_stream) {
  if (!p) return set_error(TRIOT_ERR_NULL_POINTER, "NullPointer: view 'p' is NULL");
  return expected_value_impl(out, nullptr, nullptr, d, dtype, workspace, workspace_bytes,
                             cuda_stream, with_mass != 0, p);
}

int triot_plan_describe(int op, const int64_t* const* shapes, const int64_t* iter_shape, int d,
                        int dtype, unsigned flags, const unsigned* ptr_mod32, int mode,
                        uint64_t warps, char* buf, size_t buf_len) {
  if (!shapes) return set_error(TRIOT_ERR_NULL_POINTER, "NullPointer: shapes is NULL");
  // synthetic, non-overlapping device addresses with the requested alignment
  uintptr_t base[3];
  for (int x = 0; x < 3; ++x)
    base[x] = ((uintptr_t)(x + 1) << 44) + (ptr_mod32 ? (uintptr_t)ptr_mod32[x] : 0);
  Geom g;
  int st;
  if (op == OP_EMBED)
    st = plan_embed(g, (void*)base[0], shapes[0], (const void*)base[1], shapes[1], d, dtype, flags);
  else if (op == OP_BINARY)
    st = plan_binary(g, (void*)base[0], shapes[0], (const void*)base[1], shapes[1],
                     (const void*)base[2], shapes[2], iter_shape, d, dtype, (int)flags);
  else if (op == OP_EV)
    st = plan_ev(g, (const void*)base[0], shapes[0], d, dtype);
  else if (op == OP_DOT)
    st = plan_dot(g, (const void*)base[0], shapes[0], (const void*)base[1], shapes[1], iter_shape,
                  d, dtype);
  else if (op == OP_CONV)
    st = plan_conv(g, (void*)base[2], (const void*)base[0], shapes[0], (const void*)base[1],
                   shapes[1], d, dtype);
  else if (op == OP_UPDATE)
    st = plan_update(g, (void*)base[0], shapes[0], (const void*)base[1], shapes[1],
                     (const void*)base[2], shapes[2], d, dtype);
  else
    return set_error(TRIOT_ERR_BAD_DTYPE_OR_OP, "BadOp: op = %d", op);
  if (st) return st;
  if (mode < 0 || mode > 2) return set_error(TRIOT_ERR_BAD_DTYPE_OR_OP, "BadMode: %d", mode);  // 3 = 2 with small stages
  if (!g.empty) set_decomposition(g, mode, warps ? warps : 1);
  std::string s = describe(g);
  if (buf && buf_len) {
    size_t n = s.size() < buf_len - 1 ? s.size() : buf_len - 1;
    memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
  return TRIOT_OK;
}

int triot_set_launch_policy(int mode, int blocks_per_sm) {
  if (mode < -1 || mode > 5 || blocks_per_sm < 0 || blocks_per_sm > 1024)
    return set_error(TRIOT_ERR_BAD_DTYPE_OR_OP, "BadPolicy: mode %d, blocks_per_sm %d", mode,
                     blocks_per_sm);
  // mode 5: no row windows (short odd innermost rows take flat vectors), decomposition automatic
  set_rows_enabled(mode != 5);
  if (mode == 5) mode = -1;
  g_override.mode = mode;
  g_override.bpsm = mode < 0 ? 0 : blocks_per_sm;
  g_override.q = 0;
  return TRIOT_OK;
}

int triot_fastdiv_magic(uint32_t divisor, uint32_t* mul, uint32_t* shift) {
  if (!mul || !shift) return set_error(TRIOT_ERR_NULL_POINTER, "NullPointer: output is NULL");
  if (divisor == 0) return set_error(TRIOT_ERR_BAD_SHAPE, "BadShape: divisor 0");
  fastdiv_magic(divisor, mul, shift);
  return TRIOT_OK;
}

}  // extern "C"
