// capi_host.cu -- host-buffer entry points: the ops on tensors that live in host memory,
// streamed through caller-provided device staging memory in slabs of axis 0.
//
// "a GPU speed-up is most likely when operating on a large, contiguous block of memory,
// which is allocated on the GPU or copied to the GPU in chunks, which are subsequently
// processed on the GPU".  Each slab of the output's axis-0 rows is a contiguous block of every
// row-major operand; slabs flow through a double-buffered pipeline on three streams -- host to
// device copy, the device op (the same kernels as the device entry points, on the caller's
// stream), device to host copy -- so PCIe transfers in both directions overlap each other and
// the compute.  Pinned host memory is needed for the copies to be asynchronous (pageable memory
// still works, serialised by the driver).
#include <cuda_runtime.h>
#include <stdlib.h>
#include <string.h>

#include <map>
#include <memory>
#include <mutex>
#include <utility>
#include <vector>

#include "../../include/triot.h"
#include "desc.h"
#include "plan.hpp"

namespace triot {
namespace {

int cuda_err(cudaError_t e, const char* what) {
  return set_error(TRIOT_ERR_CUDA, "CUDA: %s: %s", what, cudaGetErrorString(e));
}

// The two copy streams and the pipeline events of one (device, caller stream) pair -- created
// on first use, reused, never destroyed (one per stream the caller pipelines on).  Calls on
// different caller streams get different copy streams, so one op's device-to-host drain runs
// while another op's host-to-device feed is in flight (PCIe is full duplex); a mutex keeps
// concurrent calls on the same caller stream in order.
constexpr int kMaxSlots = 8;
struct Pipe {
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t loaded[kMaxSlots], computed[kMaxSlots], drained[kMaxSlots];
  std::mutex mu;
  bool ready = false;
};
std::mutex g_pipes_mu;
std::map<std::pair<int, cudaStream_t>, std::unique_ptr<Pipe>> g_pipes;

int pipe_for(cudaStream_t caller, Pipe** out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_err(e, "cudaGetDevice");
  std::lock_guard<std::mutex> lk(g_pipes_mu);
  std::unique_ptr<Pipe>& p = g_pipes[std::make_pair(dev, caller)];
  if (!p) p.reset(new Pipe());
  *out = p.get();
  return TRIOT_OK;
}

int pipe_init(Pipe& p) {
  if (p.ready) return TRIOT_OK;
  cudaError_t e;
  if ((e = cudaStreamCreateWithFlags(&p.h2d, cudaStreamNonBlocking)) != cudaSuccess)
    return cuda_err(e, "cudaStreamCreateWithFlags");
  if ((e = cudaStreamCreateWithFlags(&p.d2h, cudaStreamNonBlocking)) != cudaSuccess)
    return cuda_err(e, "cudaStreamCreateWithFlags");
  for (int s = 0; s < kMaxSlots; ++s) {
    cudaEvent_t* evs[3] = {&p.loaded[s], &p.computed[s], &p.drained[s]};
    for (cudaEvent_t* ev : evs)
      if ((e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming)) != cudaSuccess)
        return cuda_err(e, "cudaEventCreateWithFlags");
  }
  p.ready = true;
  return TRIOT_OK;
}

int esz_of(int dtype) { return dtype == TRIOT_F32 ? 4 : dtype == TRIOT_F64 ? 8 : 0; }

// staging slots per pipeline (the ring of chunks in flight): 6 keeps more, smaller chunks moving
// so the copy engines interleave the pipelines of concurrent calls finer (B200, the bench's four
// e2e legs: 2 slots 40.6-46.1 ms, 3: 38.5-44.1, 4: 40.3-46.7, 6: 36.9-38.2 ms per step,
// profiles/r02_e2e_slots2.jsonl); TRIOT_HOST_SLOTS overrides it for A/B runs (tools/e2e_probe.py)
int host_slots() {
  static int n = [] {
    const char* e = getenv("TRIOT_HOST_SLOTS");
    int v = e ? atoi(e) : 6;
    return v < 2 ? 2 : v > kMaxSlots ? kMaxSlots : v;
  }();
  return n;
}

// Elements of one index of axis k: prod_{j > k} shape[j].
uint64_t sub_elems(const int64_t* shape, int d, int k) {
  uint64_t n = 1;
  for (int j = k + 1; j < d; ++j) n *= (uint64_t)shape[j];
  return n;
}

// The generic pipeline.  A chunk is a prefix tuple (t_0 .. t_{k-1}) of the output plus a range
// [a, a + rows) of axis k: a contiguous block of the row-major output and of every input that
// contains the prefix (inputs that do not -- an embed's src outside the prefix -- contribute an
// empty slab).  k is the first axis whose sub-rows let two slots of one chunk fit the staging.
// `op(out_sub_shape, in_sub_shapes, dev_in[], dev_out, dsub)` enqueues the device op on the
// caller's stream for the chunk (shapes of dsub = d - k dimensions).
template <typename OpFn>
int run_pipeline(void* out_h, const int64_t* out_shape, int nin, const void* const* in_h,
                 const int64_t* const* in_shape, int d, int esz, void* staging,
                 size_t staging_bytes, cudaStream_t compute, OpFn op) {
  Pipe* pp;
  int st = pipe_for(compute, &pp);
  if (st) return st;
  Pipe& P = *pp;
  std::lock_guard<std::mutex> lk(P.mu);
  if ((st = pipe_init(P))) return st;
  const int NSL = host_slots();
  const uint64_t slot_bytes = (staging_bytes / (uint64_t)NSL) & ~255ull;  // slots 256-B aligned
  const uint64_t pad = 256 * (uint64_t)(nin + 1);
  // choose the chunk axis k and the rows per chunk
  int k = 0;
  uint64_t per_row = 0;
  for (; k < d; ++k) {
    per_row = sub_elems(out_shape, d, k) * (uint64_t)esz;
    for (int i = 0; i < nin; ++i) per_row += sub_elems(in_shape[i], d, k) * (uint64_t)esz;
    if (slot_bytes > pad && per_row <= slot_bytes - pad) break;
  }
  if (k == d)
    return set_error(TRIOT_ERR_WORKSPACE,
                     "Workspace: %zu staging bytes cannot hold two chunks of one element",
                     staging_bytes);
  const uint64_t nk = (uint64_t)out_shape[k];
  uint64_t rows = (slot_bytes - pad) / per_row;
  if (rows > nk) rows = nk ? nk : 1;
  const int dsub = d - k;
  const uint64_t out_row = sub_elems(out_shape, d, k) * (uint64_t)esz;
  uint64_t in_row[TRIOT_MAXT];
  for (int i = 0; i < nin; ++i) in_row[i] = sub_elems(in_shape[i], d, k) * (uint64_t)esz;
  auto align = [](uint64_t x) { return (x + 255) & ~255ull; };
  char* dev_out[kMaxSlots];
  char* dev_in[kMaxSlots][TRIOT_MAXT];
  for (int s = 0; s < NSL; ++s) {
    char* q = (char*)staging + (size_t)s * slot_bytes;
    dev_out[s] = q;
    q += align(rows * out_row);
    for (int i = 0; i < nin; ++i) {
      dev_in[s][i] = q;
      q += align(rows * in_row[i]);
    }
  }
  cudaError_t e;
  // the first copies must not overtake work already queued on the caller's stream
  if ((e = cudaEventRecord(P.computed[0], compute)) != cudaSuccess) return cuda_err(e, "record");
  if ((e = cudaStreamWaitEvent(P.h2d, P.computed[0], 0)) != cudaSuccess)
    return cuda_err(e, "wait");
  if ((e = cudaStreamWaitEvent(P.d2h, P.computed[0], 0)) != cudaSuccess)
    return cuda_err(e, "wait");
  uint64_t prefix[TRIOT_MAXD] = {0};
  uint64_t npre = 1;
  for (int j = 0; j < k; ++j) npre *= (uint64_t)out_shape[j];
  uint64_t chunk = 0;
  for (uint64_t pi = 0; pi < npre; ++pi) {
    // Horner offsets of the prefix (in units of axis-k rows) in the output and each input
    uint64_t out_base = 0, in_base[TRIOT_MAXT];
    bool in_ok[TRIOT_MAXT];
    for (int j = 0; j < k; ++j) out_base = out_base * (uint64_t)out_shape[j] + prefix[j];
    out_base *= nk;
    for (int i = 0; i < nin; ++i) {
      uint64_t b = 0;
      in_ok[i] = true;
      for (int j = 0; j < k; ++j) {
        if (prefix[j] >= (uint64_t)in_shape[i][j]) in_ok[i] = false;
        b = b * (uint64_t)in_shape[i][j] + prefix[j];
      }
      in_base[i] = b * (uint64_t)in_shape[i][k];
    }
    for (uint64_t a = 0; a < nk; a += rows, ++chunk) {
      const int s = (int)(chunk % (uint64_t)NSL);
      const uint64_t r = a + rows <= nk ? rows : nk - a;
      if (chunk >= (uint64_t)NSL) {  // slot reuse: its last chunk's inputs consumed, output drained
        if ((e = cudaStreamWaitEvent(P.h2d, P.computed[s], 0)) != cudaSuccess)
          return cuda_err(e, "wait");
        if ((e = cudaStreamWaitEvent(compute, P.drained[s], 0)) != cudaSuccess)
          return cuda_err(e, "wait");
      }
      int64_t in_sub[TRIOT_MAXT][TRIOT_MAXD];
      for (int i = 0; i < nin; ++i) {
        const uint64_t ext = (uint64_t)in_shape[i][k];
        uint64_t ir = (!in_ok[i] || a >= ext) ? 0 : (r < ext - a ? r : ext - a);
        in_sub[i][0] = (int64_t)ir;
        for (int j = 1; j < dsub; ++j) in_sub[i][j] = in_shape[i][k + j];
        if (ir) {
          e = cudaMemcpyAsync(dev_in[s][i], (const char*)in_h[i] + (in_base[i] + a) * in_row[i],
                              ir * in_row[i], cudaMemcpyHostToDevice, P.h2d);
          if (e != cudaSuccess) return cuda_err(e, "cudaMemcpyAsync H2D");
        }
      }
      if ((e = cudaEventRecord(P.loaded[s], P.h2d)) != cudaSuccess) return cuda_err(e, "record");
      if ((e = cudaStreamWaitEvent(compute, P.loaded[s], 0)) != cudaSuccess)
        return cuda_err(e, "wait");
      int64_t out_sub[TRIOT_MAXD];
      out_sub[0] = (int64_t)r;
      for (int j = 1; j < dsub; ++j) out_sub[j] = out_shape[k + j];
      const int64_t* in_sub_p[TRIOT_MAXT];
      for (int i = 0; i < nin; ++i) in_sub_p[i] = in_sub[i];
      if ((st = op(out_sub, in_sub_p, dev_in[s], dev_out[s], dsub))) return st;
      if ((e = cudaEventRecord(P.computed[s], compute)) != cudaSuccess)
        return cuda_err(e, "record");
      if ((e = cudaStreamWaitEvent(P.d2h, P.computed[s], 0)) != cudaSuccess)
        return cuda_err(e, "wait");
      e = cudaMemcpyAsync((char*)out_h + (out_base + a) * out_row, dev_out[s], r * out_row,
                          cudaMemcpyDeviceToHost, P.d2h);
      if (e != cudaSuccess) return cuda_err(e, "cudaMemcpyAsync D2H");
      if ((e = cudaEventRecord(P.drained[s], P.d2h)) != cudaSuccess)
        return cuda_err(e, "record");
    }
    for (int j = k - 1; j >= 0; --j) {  // Alg 3 on the prefix
      if (++prefix[j] < (uint64_t)out_shape[j]) break;
      prefix[j] = 0;
    }
  }
  // the caller's stream completes only when the last chunk has landed in host memory
  for (int s = 0; s < NSL; ++s)
    if (chunk > (uint64_t)s)
      if ((e = cudaStreamWaitEvent(compute, P.drained[s], 0)) != cudaSuccess)
        return cuda_err(e, "wait");
  return TRIOT_OK;
}

}  // namespace
}  // namespace triot

using namespace triot;

extern "C" {

int triot_embed_host(void* dst, const int64_t* dst_shape, const void* src,
                     const int64_t* src_shape, int d, int dtype, unsigned flags, void* staging,
                     size_t staging_bytes, void* cuda_stream) {
  // validate exactly as the device entry point would (host pointers stand in for the data)
  Geom g;
  int st = plan_embed(g, dst, dst_shape, src, src_shape, d, dtype, flags);
  if (st) return st;
  if (g.empty) return TRIOT_OK;
  if (!staging) return set_error(TRIOT_ERR_WORKSPACE, "Workspace: staging is NULL");
  const int esz = esz_of(dtype);
  const void* ins[1] = {src};
  const int64_t* ishp[1] = {src_shape};
  const bool region = (flags & TRIOT_EMBED_REGION_ONLY) != 0;
  cudaStream_t cs = (cudaStream_t)cuda_stream;
  if (region) {
    // region-only writes part of dst: bring the dst slab in first so the rest is preserved
    return set_error(TRIOT_ERR_BAD_DTYPE_OR_OP,
                     "BadFlags: triot_embed_host supports TRIOT_EMBED_FULL only");
  }
  return run_pipeline(dst, dst_shape, 1, ins, ishp, d, esz, staging, staging_bytes, cs,
                      [&](const int64_t* out_sub, const int64_t* const* in_sub, char* const* din,
                          char* dout, int dsub) -> int {
                        return triot_embed(dout, out_sub, din[0], in_sub[0], dsub, dtype, flags,
                                           cs);
                      });
}

int triot_expected_value_host(double* out, const void* p, const int64_t* shape,
                              const int64_t* offset, int d, int dtype, int with_mass,
                              void* staging, size_t staging_bytes, void* cuda_stream) {
  Geom g;
  int st = plan_ev(g, p, shape, d, dtype);
  if (st) return st;
  if (!out) return set_error(TRIOT_ERR_NULL_POINTER, "NullPointer: out is NULL");
  if (!staging) return set_error(TRIOT_ERR_WORKSPACE, "Workspace: staging is NULL");
  if (((uintptr_t)staging) % 256)
    return set_error(TRIOT_ERR_MISALIGNED, "Misaligned: staging is not 256-byte aligned");
  const int esz = esz_of(dtype);
  const int nout = d + (with_mass ? 1 : 0);
  size_t ws_bytes = 0;
  if ((st = triot_expected_value_workspace_size(shape, d, dtype, &ws_bytes))) return st;
  auto align = [](uint64_t x) { return (x + 255) & ~255ull; };
  cudaStream_t cs = (cudaStream_t)cuda_stream;
  Pipe* pp;
  if ((st = pipe_for(cs, &pp))) return st;
  Pipe& P = *pp;
  std::lock_guard<std::mutex> lk(P.mu);
  if ((st = pipe_init(P))) return st;
  // staging: [workspace][final: nout][rows: nchunk x nout][slot 0][slot 1]
  const uint64_t fixed = align(ws_bytes) + align((uint64_t)nout * 8);
  if (staging_bytes <= fixed + 512)
    return set_error(TRIOT_ERR_WORKSPACE, "Workspace: %zu staging bytes, need > %llu", staging_bytes,
                     (unsigned long long)(fixed + 512));
  if (offset)
    for (int j = 0; j < d; ++j)
      if (offset[j] < 0 || offset[j] + shape[j] > (int64_t)(1ll << 53))
        return set_error(TRIOT_ERR_BAD_SHAPE, "BadShape: offset[%d] = %lld outside [0, 2^53)", j,
                         (long long)offset[j]);
  if (g.empty) {  // empty sums: zeros
    double* fin0 = (double*)((char*)staging + align(ws_bytes));
    cudaError_t e0 = cudaMemsetAsync(fin0, 0, (size_t)nout * 8, cs);
    if (e0 == cudaSuccess)
      e0 = cudaMemcpyAsync(out, fin0, (size_t)nout * 8, cudaMemcpyDeviceToHost, cs);
    if (e0 != cudaSuccess) return cuda_err(e0, "empty expected value");
    clear_error();
    return TRIOT_OK;
  }
  // choose the chunk axis k (the first whose single index fits a slot, with room for the rows)
  int k = 0;
  uint64_t rows = 0, nchunk = 0, row_bytes = 0, npre = 1;
  for (; k < d; ++k) {
    row_bytes = sub_elems(shape, d, k) * (uint64_t)esz;
    const uint64_t nk = (uint64_t)shape[k];
    // rows per chunk r: 2 * align(r row_bytes) + align(chunks(r) * nout * 8) <= avail
    const uint64_t avail = staging_bytes - fixed;
    uint64_t r = (avail / 2) / (row_bytes ? row_bytes : 1);
    if (r > nk) r = nk;
    while (r >= 1) {
      const uint64_t nc = npre * ((nk + r - 1) / r);
      if (2 * align(r * row_bytes) + align(nc * (uint64_t)nout * 8) <= avail) break;
      r = r > 1 ? r / 2 : 0;
    }
    if (r >= 1) {
      rows = r;
      nchunk = npre * ((nk + r - 1) / r);
      break;
    }
    npre *= nk;
  }
  if (k == d)
    return set_error(TRIOT_ERR_WORKSPACE, "Workspace: %zu staging bytes cannot hold two chunks",
                     staging_bytes);
  char* base = (char*)staging;
  void* ws = base;
  double* fin = (double*)(base + align(ws_bytes));
  double* rowsbuf = (double*)(base + fixed);
  char* slot[2];
  slot[0] = base + fixed + align(nchunk * (uint64_t)nout * 8);
  slot[1] = slot[0] + align(rows * row_bytes);
  cudaError_t e;
  // the workspace must start zeroed (the reduction leaves it zeroed afterwards)
  if ((e = cudaMemsetAsync(ws, 0, ws_bytes, cs)) != cudaSuccess) return cuda_err(e, "memset");
  if ((e = cudaEventRecord(P.computed[0], cs)) != cudaSuccess) return cuda_err(e, "record");
  if ((e = cudaStreamWaitEvent(P.h2d, P.computed[0], 0)) != cudaSuccess) return cuda_err(e, "wait");
  const uint64_t nk = (uint64_t)shape[k];
  int64_t csh[TRIOT_MAXD], off[TRIOT_MAXD];
  uint64_t prefix[TRIOT_MAXD] = {0};
  uint64_t chunk = 0;
  for (uint64_t pi = 0; pi < npre; ++pi) {
    uint64_t pbase = 0;  // Horner of the prefix, in units of axis-k index rows
    for (int j = 0; j < k; ++j) pbase = pbase * (uint64_t)shape[j] + prefix[j];
    pbase *= nk;
    for (uint64_t a = 0; a < nk; a += rows, ++chunk) {
      const int s = (int)(chunk & 1);
      const uint64_t r = a + rows <= nk ? rows : nk - a;
      if (chunk >= 2)  // the slot's previous chunk has been consumed
        if ((e = cudaStreamWaitEvent(P.h2d, P.computed[s], 0)) != cudaSuccess)
          return cuda_err(e, "wait");
      e = cudaMemcpyAsync(slot[s], (const char*)p + (pbase + a) * row_bytes, r * row_bytes,
                          cudaMemcpyHostToDevice, P.h2d);
      if (e != cudaSuccess) return cuda_err(e, "cudaMemcpyAsync H2D");
      if ((e = cudaEventRecord(P.loaded[s], P.h2d)) != cudaSuccess) return cuda_err(e, "record");
      if ((e = cudaStreamWaitEvent(cs, P.loaded[s], 0)) != cudaSuccess) return cuda_err(e, "wait");
      // the chunk as a d-dimensional block (1, .., 1, r, s_{k+1}, ..) at (prefix, a, 0, ..)
      for (int j = 0; j < d; ++j) {
        csh[j] = j < k ? 1 : j == k ? (int64_t)r : shape[j];
        off[j] = (offset ? offset[j] : 0) + (j < k ? (int64_t)prefix[j] : j == k ? (int64_t)a : 0);
      }
      if ((st = triot_expected_value_offset(rowsbuf + chunk * (uint64_t)nout, slot[s], csh, off, d,
                                            dtype, with_mass, ws, ws_bytes, cs)))
        return st;
      if ((e = cudaEventRecord(P.computed[s], cs)) != cudaSuccess) return cuda_err(e, "record");
    }
    for (int j = k - 1; j >= 0; --j) {  // Alg 3 on the prefix
      if (++prefix[j] < (uint64_t)shape[j]) break;
      prefix[j] = 0;
    }
  }
  if ((st = triot_sum_rows(fin, rowsbuf, (int64_t)nchunk, nout, cs))) return st;
  e = cudaMemcpyAsync(out, fin, (size_t)nout * 8, cudaMemcpyDeviceToHost, cs);
  if (e != cudaSuccess) return cuda_err(e, "cudaMemcpyAsync D2H");
  clear_error();
  return TRIOT_OK;
}

int triot_apply_binary_host(void* c, const void* a, const int64_t* a_shape, const void* b,
                            const int64_t* b_shape, const int64_t* iter_shape, int d, int dtype,
                            int op, void* staging, size_t staging_bytes, void* cuda_stream) {
  // host variant: c is dense in the iteration shape
  Geom g;
  int st = plan_binary(g, c, nullptr, a, a_shape, b, b_shape, iter_shape, d, dtype, op);
  if (st) return st;
  if (g.empty) return TRIOT_OK;
  if (!staging) return set_error(TRIOT_ERR_WORKSPACE, "Workspace: staging is NULL");
  int64_t it[TRIOT_MAXD];
  for (int k = 0; k < d; ++k)
    it[k] = iter_shape ? iter_shape[k] : (a_shape[k] < b_shape[k] ? a_shape[k] : b_shape[k]);
  const int esz = esz_of(dtype);
  const void* ins[2] = {a, b};
  const int64_t* ishp[2] = {a_shape, b_shape};
  cudaStream_t cs = (cudaStream_t)cuda_stream;
  return run_pipeline(c, it, 2, ins, ishp, d, esz, staging, staging_bytes, cs,
                      [&](const int64_t* out_sub, const int64_t* const* in_sub, char* const* din,
                          char* dout, int dsub) -> int {
                        return triot_apply_binary(dout, out_sub, din[0], in_sub[0], din[1],
                                                  in_sub[1], out_sub, dsub, dtype, op, cs);
                      });
}

}  // extern "C"
