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
#include <string.h>

#include <mutex>
#include <vector>

#include "../../include/triot.h"
#include "desc.h"
#include "plan.hpp"

namespace triot {
namespace {

int cuda_err(cudaError_t e, const char* what) {
  return set_error(TRIOT_ERR_CUDA, "CUDA: %s: %s", what, cudaGetErrorString(e));
}

// Per-device pool of the two copy streams and the pipeline events (created once, reused;
// guarded by a mutex: one host-buffer call at a time per device).
struct Pipe {
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t loaded[2], computed[2], drained[2];
  std::mutex mu;
  bool ready = false;
};
Pipe g_pipes[64];

int pipe_for(Pipe** out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_err(e, "cudaGetDevice");
  if (dev < 0 || dev >= 64) return set_error(TRIOT_ERR_CUDA, "CUDA: device id %d", dev);
  Pipe& p = g_pipes[dev];
  *out = &p;
  return TRIOT_OK;
}

int pipe_init(Pipe& p) {
  if (p.ready) return TRIOT_OK;
  cudaError_t e;
  if ((e = cudaStreamCreateWithFlags(&p.h2d, cudaStreamNonBlocking)) != cudaSuccess)
    return cuda_err(e, "cudaStreamCreateWithFlags");
  if ((e = cudaStreamCreateWithFlags(&p.d2h, cudaStreamNonBlocking)) != cudaSuccess)
    return cuda_err(e, "cudaStreamCreateWithFlags");
  for (int s = 0; s < 2; ++s) {
    cudaEvent_t* evs[3] = {&p.loaded[s], &p.computed[s], &p.drained[s]};
    for (cudaEvent_t* ev : evs)
      if ((e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming)) != cudaSuccess)
        return cuda_err(e, "cudaEventCreateWithFlags");
  }
  p.ready = true;
  return TRIOT_OK;
}

uint64_t row_elems(const int64_t* shape, int d) {
  uint64_t n = 1;
  for (int k = 1; k < d; ++k) n *= (uint64_t)shape[k];
  return n;
}

// A slab of `rows` rows starting at row `lo` of a tensor of `shape`, clipped to its extent.
struct Slab {
  uint64_t lo, rows;
};
Slab clip(uint64_t lo, uint64_t rows, int64_t extent0) {
  uint64_t e = (uint64_t)extent0;
  if (lo >= e) return Slab{lo, 0};
  return Slab{lo, rows < e - lo ? rows : e - lo};
}

int esz_of(int dtype) { return dtype == TRIOT_F32 ? 4 : dtype == TRIOT_F64 ? 8 : 0; }

// The generic pipeline.  `nin` inputs are copied in (their slabs of the output's rows), the op
// runs on the device slabs, the output slab is copied out.  `op(slot, rows_out, in_rows[],
// dev_in[], dev_out)` enqueues the device op on `compute`.
template <typename OpFn>
int run_pipeline(void* out_h, const int64_t* out_shape, int nin, const void* const* in_h,
                 const int64_t* const* in_shape, int d, int esz, void* staging,
                 size_t staging_bytes, cudaStream_t compute, OpFn op) {
  Pipe* pp;
  int st = pipe_for(&pp);
  if (st) return st;
  Pipe& P = *pp;
  std::lock_guard<std::mutex> lk(P.mu);
  if ((st = pipe_init(P))) return st;
  const uint64_t n0 = (uint64_t)out_shape[0];
  const uint64_t out_row = row_elems(out_shape, d) * (uint64_t)esz;
  uint64_t in_row[TRIOT_MAXT];
  uint64_t per_row = out_row;
  for (int i = 0; i < nin; ++i) {
    in_row[i] = row_elems(in_shape[i], d) * (uint64_t)esz;
    per_row += in_row[i];
  }
  // two slots, each holding a slab of every operand, 256-B aligned pieces
  const uint64_t slot_bytes = staging_bytes / 2;
  uint64_t rows = per_row ? (slot_bytes - 256 * (uint64_t)(nin + 1)) / per_row : n0;
  if (rows < 1 || slot_bytes < 256 * (uint64_t)(nin + 1) + per_row)
    return set_error(TRIOT_ERR_WORKSPACE,
                     "Workspace: %zu staging bytes cannot hold two slabs of one row (%llu B)",
                     staging_bytes, (unsigned long long)(2 * (per_row + 256 * (nin + 1))));
  if (rows > n0) rows = n0 ? n0 : 1;
  auto align = [](uint64_t x) { return (x + 255) & ~255ull; };
  char* slot_base[2] = {(char*)staging, (char*)staging + slot_bytes};
  char* dev_out[2];
  char* dev_in[2][TRIOT_MAXT];
  for (int s = 0; s < 2; ++s) {
    char* q = slot_base[s];
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
  uint64_t chunk = 0;
  for (uint64_t lo = 0; lo < n0; lo += rows, ++chunk) {
    const int s = (int)(chunk & 1);
    const uint64_t r = lo + rows <= n0 ? rows : n0 - lo;
    // slot reuse: the inputs of chunk-2 were consumed by its compute, its output drained
    if (chunk >= 2) {
      if ((e = cudaStreamWaitEvent(P.h2d, P.computed[s], 0)) != cudaSuccess)
        return cuda_err(e, "wait");
      if ((e = cudaStreamWaitEvent(compute, P.drained[s], 0)) != cudaSuccess)
        return cuda_err(e, "wait");
    }
    uint64_t in_rows[TRIOT_MAXT];
    for (int i = 0; i < nin; ++i) {
      Slab sl = clip(lo, r, in_shape[i][0]);
      in_rows[i] = sl.rows;
      if (sl.rows) {
        e = cudaMemcpyAsync(dev_in[s][i], (const char*)in_h[i] + sl.lo * in_row[i],
                            sl.rows * in_row[i], cudaMemcpyHostToDevice, P.h2d);
        if (e != cudaSuccess) return cuda_err(e, "cudaMemcpyAsync H2D");
      }
    }
    if ((e = cudaEventRecord(P.loaded[s], P.h2d)) != cudaSuccess) return cuda_err(e, "record");
    if ((e = cudaStreamWaitEvent(compute, P.loaded[s], 0)) != cudaSuccess)
      return cuda_err(e, "wait");
    if ((st = op(lo, r, in_rows, dev_in[s], dev_out[s]))) return st;
    if ((e = cudaEventRecord(P.computed[s], compute)) != cudaSuccess)
      return cuda_err(e, "record");
    if ((e = cudaStreamWaitEvent(P.d2h, P.computed[s], 0)) != cudaSuccess)
      return cuda_err(e, "wait");
    if (out_h) {
      e = cudaMemcpyAsync((char*)out_h + lo * out_row, dev_out[s], r * out_row,
                          cudaMemcpyDeviceToHost, P.d2h);
      if (e != cudaSuccess) return cuda_err(e, "cudaMemcpyAsync D2H");
    }
    if ((e = cudaEventRecord(P.drained[s], P.d2h)) != cudaSuccess) return cuda_err(e, "record");
  }
  // the caller's stream completes only when the last slab has landed in host memory
  for (int s = 0; s < 2; ++s)
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
                      [&](uint64_t lo, uint64_t rows, const uint64_t* in_rows, char* const* din,
                          char* dout) -> int {
                        int64_t ds[TRIOT_MAXD], ss[TRIOT_MAXD];
                        for (int k = 0; k < d; ++k) {
                          ds[k] = dst_shape[k];
                          ss[k] = src_shape[k];
                        }
                        ds[0] = (int64_t)rows;
                        ss[0] = (int64_t)in_rows[0];
                        (void)lo;
                        return triot_embed(dout, ds, din[0], ss, d, dtype, flags, cs);
                      });
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
                      [&](uint64_t lo, uint64_t rows, const uint64_t* in_rows, char* const* din,
                          char* dout) -> int {
                        int64_t as[TRIOT_MAXD], bs[TRIOT_MAXD], is[TRIOT_MAXD];
                        for (int k = 0; k < d; ++k) {
                          as[k] = a_shape[k];
                          bs[k] = b_shape[k];
                          is[k] = it[k];
                        }
                        as[0] = (int64_t)in_rows[0];
                        bs[0] = (int64_t)in_rows[1];
                        is[0] = (int64_t)rows;
                        (void)lo;
                        return triot_apply_binary(dout, is, din[0], as, din[1], bs, is, d, dtype,
                                                  op, cs);
                      });
}

}  // extern "C"
