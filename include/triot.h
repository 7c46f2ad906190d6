/*
 * triot.h -- C-ABI of the B200 (sm_100a) TRIOT hot path.
 *
 * TRIOT = "template-recursive iteration over tensors" (Heyl & Serang, arXiv 1608.00099; the
 * paper text is cited as P:<line>).  The hot path is tuple-indexed iteration over a counter
 * shape: for every index tuple t of the counter, each tensor's flat offset is computed by
 * Horner's rule over that tensor's OWN shape (Alg 2, applied per tensor at
 * P:217), then an operation that may read t is applied (Alg 10).  This library
 * exports the three instances of that path the build targets:
 *
 *   triot_embed            zero-padded embedding (or crop) of one tensor into another
 *                          (the Benchmark-1 body "xV = yV")
 *   triot_apply_binary     c[t] = a[t] OP b[t] over tensors of different shapes
 *                          (Alg 9 apply_tensors; PMF products P:613)
 *   triot_expected_value   m_k = sum_t t_k * p[t], the index-weighted reduction
 *                          (Alg 11; "expected value computation")
 *
 * Conventions shared by every entry point:
 *   - Layout: every tensor is a dense, row-major ("as used in the C programming language",
 *     P:50) contiguous buffer plus a host array `const int64_t shape[d]`.  One d per call.
 *     Shapes are read during the call and not retained.
 *   - Dimension: 1 <= d <= triot_max_dimension() (= 16).  The paper fixes a compile-time
 *     maximum (MAX_TENSOR_DIMENSION) and dispatches a runtime d onto compile-time
 *     instances (Alg 7); here the instances are sm_100a kernels for D = 1..16.
 *   - Ownership: every data pointer (dst, src, a, b, c, p, means, workspace) is a DEVICE
 *     pointer owned by the caller.  The library never allocates or frees device memory.
 *   - Extents may be 0 (empty tensors).  Elements are float32 (TRIOT_F32) or float64
 *     (TRIOT_F64); every tensor of one call has the same dtype.  Data pointers must be aligned
 *     to the element size; wider (up to 32-byte) accesses are chosen at run time.
 *   - Checking: one up-front check over shapes, never per element.  Validation errors
 *     return synchronously before anything is enqueued; nothing is written.
 *   - Asynchrony: work is enqueued on `cuda_stream` (a cudaStream_t passed as void*; NULL =
 *     the legacy default stream) and the call returns.  Device faults surface at the caller's
 *     next synchronisation.  Launch failures return TRIOT_ERR_CUDA.
 *   - Errors: return codes only (never exceptions across the ABI).  triot_last_error()
 *     returns a thread-local message naming the tensor and axis (the vocabulary of the
 *     paper's check_tensor_pack_bounds).
 *   - Aliasing: the written tensor must not overlap any input (the paper relies on
 *     __restrict), except exact in-place binary ops (see triot_apply_binary).
 *   - Thread safety: stateless apart from cached per-device attributes; callable from
 *     several host threads on different streams.
 *
 * This header does not include any CUDA header.
 */
#ifndef TRIOT_H_
#define TRIOT_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define TRIOT_API __attribute__((visibility("default")))
#else
#define TRIOT_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { TRIOT_F32 = 0, TRIOT_F64 = 1 } triot_dtype;

typedef enum { TRIOT_ADD = 0, TRIOT_SUB = 1, TRIOT_MUL = 2, TRIOT_DIV = 3 } triot_binop;

enum {
  TRIOT_EMBED_FULL = 0u,        /* write every element of dst (zeros outside src)            */
  TRIOT_EMBED_REGION_ONLY = 1u  /* write only t < min(src_shape, dst_shape)                  */
};

typedef enum {
  TRIOT_OK = 0,
  TRIOT_ERR_NULL_POINTER = 1,          /* non-empty tensor with NULL data, or NULL shape/out   */
  TRIOT_ERR_UNSUPPORTED_DIMENSION = 2, /* d < 1 || d > triot_max_dimension()                   */
  TRIOT_ERR_BAD_SHAPE = 3,             /* negative extent, or a tensor of >= 2^62 bytes        */
  TRIOT_ERR_AXIS_OUT_OF_BOUNDS = 4,    /* iteration shape exceeds an operand on some axis      */
  TRIOT_ERR_BAD_DTYPE_OR_OP = 5,       /* unknown dtype, op or flag bits                       */
  TRIOT_ERR_MISALIGNED = 6,            /* data pointer not aligned to its element size         */
  TRIOT_ERR_ALIASING = 7,              /* output overlaps an input (other than exact in-place) */
  TRIOT_ERR_WORKSPACE = 8,             /* workspace NULL or smaller than the queried size      */
  TRIOT_ERR_CUDA = 9                   /* a CUDA call failed; detail in triot_last_error()     */
} triot_status;

/* 16: the largest d with a compiled instance (the paper's MAX_TENSOR_DIMENSION). */
TRIOT_API int triot_max_dimension(void);

/* Static string for a status code ("TRIOT_OK", "TRIOT_ERR_ALIASING", ...). Never NULL. */
TRIOT_API const char* triot_status_string(int status);

/* Thread-local detail of the last non-OK return on this thread (e.g. "AxisOutOfBounds: tensor
 * 'a' axis 2: iteration extent 7 > tensor extent 5").  Empty string after success. */
TRIOT_API const char* triot_last_error(void);

/*
 * triot_embed -- zero-padded embedding ("copying data from one tensor to another larger,
 * zero padded tensor"; "zero padding a tensor to perform convolution via the
 * multidimensional fast Fourier transform"), i.e. apply_tensors with body "xV = yV"
 * iterated over dst's shape.
 *
 *   flags == TRIOT_EMBED_FULL:        for every t in prod[0, dst_shape[k]):
 *                                       dst[t] = (t_k < src_shape[k] for all k) ? src[t] : +0.0
 *   flags == TRIOT_EMBED_REGION_ONLY: for every t in prod[0, min(src_shape[k], dst_shape[k])):
 *                                       dst[t] = src[t]; other elements of dst are not written.
 *
 * src may be larger than dst on any axis (a crop, the paper's Benchmark 1) and
 * smaller on others (pad).  Elements are moved as raw bits (NaN payloads, -0.0, subnormals
 * survive); the padding is the all-zero bit pattern (+0.0).
 *   dst, src:   device pointers, dense row-major, dtype `dtype`; must not overlap.
 *   dst_shape, src_shape: host arrays of d extents.
 * Empty dst: no-op.  Empty src with FULL: dst becomes all +0.0.
 */
TRIOT_API int triot_embed(void* dst, const int64_t* dst_shape,
                const void* src, const int64_t* src_shape,
                int d, int dtype, unsigned flags, void* cuda_stream);

/*
 * triot_apply_binary -- element-wise op over tensors of different shapes (Alg 9 apply_tensors,
 * only the destination is written; "the product of two or more probability mass
 * functions with varying support"):
 *
 *   for every t in prod[0, iter_shape[k]):   c[t] = a[t] OP b[t]
 *
 * where each of a, b, c is indexed by its OWN shape.  OP is IEEE-754 round-to-nearest
 * with a single rounding (no contraction, no flush-to-zero).
 *   iter_shape == NULL: the element-wise minimum of a_shape and b_shape (the paper leaves the
 *                       iteration shape to the caller, "assumes x has smaller shape").
 *   c_shape == NULL:    c is dense in iter_shape.  Otherwise c_shape >= iter_shape per axis and
 *                       the elements of c outside iter_shape are left untouched.
 * iter_shape must not exceed a_shape, b_shape or c_shape on any axis
 * (TRIOT_ERR_AXIS_OUT_OF_BOUNDS, naming the tensor and axis).
 * c must not overlap a or b, except c == a (or c == b) with identical shape and iter_shape equal
 * to that shape (pure in-place; the aliasing-safe idiom of P:601).
 */
TRIOT_API int triot_apply_binary(void* c, const int64_t* c_shape,
                       const void* a, const int64_t* a_shape,
                       const void* b, const int64_t* b_shape,
                       const int64_t* iter_shape, int d, int dtype, int op, void* cuda_stream);

/*
 * triot_expected_value_workspace_size -- bytes of device workspace triot_expected_value needs for
 * this shape.  The workspace must be zero-filled ONCE when allocated; every call leaves its
 * completion ticket at zero again, so no per-call memset is needed.  One workspace per
 * concurrently running stream.
 */
TRIOT_API int triot_expected_value_workspace_size(const int64_t* shape, int d, int dtype, size_t* bytes);

/*
 * triot_expected_value -- Alg 11 with a single tensor:
 *
 *   means[k] = sum over t in prod[0, shape[j]) of  t_k * p[t],     k = 0..d-1
 *
 * accumulated in fp64 for both dtypes (Alg 11's Vector<double> result), with 0-based
 * tuple coordinates as weights (counter[k]) and NO normalisation by sum(p) (Alg 11 never
 * divides).  The result is deterministic run to run on one device (fixed grid, ordered final
 * sum); it matches the correctly rounded sum within 1e-12 relative per component.
 *   means:     device pointer to d doubles (written by the kernel).
 *   p:         device pointer, dense row-major, dtype `dtype`.
 *   workspace: device pointer of >= triot_expected_value_workspace_size bytes, zeroed once.
 * Empty p (some extent 0): means are all 0.0.
 */
TRIOT_API int triot_expected_value(double* means, const void* p, const int64_t* shape, int d, int dtype,
                         void* workspace, size_t workspace_bytes, void* cuda_stream);

/*
 * triot_expected_value_mass -- as triot_expected_value, and additionally out[d] = sum_t p[t]
 * (fp64): out must hold d + 1 doubles.  The mass is the term that amalgamates slab-sharded
 * pre-results: a rank holding axis-0 rows [o, o + n) of a larger p adds o * out[d] to
 * its out[0] before the cross-rank sum (paper_1608_00099_b200/parallel.py).
 */
TRIOT_API int triot_expected_value_mass(double* out, const void* p, const int64_t* shape, int d,
                                        int dtype, void* workspace, size_t workspace_bytes,
                                        void* cuda_stream);

/* ---- blocks of a larger PMF and the amalgamation of pre-results ----------------
 *
 * P:607 splits the outer loops across processors: "each thread computes its own pre-result and
 * these pre-results are amalgamated".  triot_expected_value_offset computes Alg 11
 * for a block p of a larger PMF whose element t sits at the global tuple offset + t:
 *   out[j] = sum_t (offset[j] + t_j) p[t]  (j < d),  out[d] = sum_t p[t] if with_mass,
 * evaluated on the device as m_j + offset[j] * mass (one rounding).  offset: host array of d
 * entries in [0, 2^53] (NULL = zeros); everything else as triot_expected_value (device buffers,
 * the same workspace, asynchronous on cuda_stream).  Summing the outputs of the blocks of a
 * partition with triot_sum_rows gives the expected value of the whole PMF.
 */
TRIOT_API int triot_expected_value_offset(double* out, const void* p, const int64_t* shape,
                                          const int64_t* offset, int d, int dtype, int with_mass,
                                          void* workspace, size_t workspace_bytes,
                                          void* cuda_stream);

/* out[j] = sum_{r < nrows} rows[r * ncols + j] for j < ncols, rows added in order (deterministic):
 * the amalgamation step.  Device buffers (out must not overlap rows), asynchronous on
 * cuda_stream; nrows == 0 writes zeros. */
TRIOT_API int triot_sum_rows(double* out, const double* rows, int64_t nrows, int64_t ncols,
                             void* cuda_stream);

/* ---- host-buffer entry points: chunked streaming through device staging memory --------
 *
 * "a GPU speed-up is most likely when operating on a large, contiguous block of memory,
 * which is allocated on the GPU or copied to the GPU in chunks, which are subsequently processed
 * on the GPU".  These take HOST pointers (pinned memory for full overlap), split the output's
 * axis 0 into slabs that fit half of the caller's device `staging` buffer, and pipeline
 * host->device copy / the device op / device->host copy of consecutive slabs on three streams.
 * Results are bit-identical to the device entry points.  The call is asynchronous with respect
 * to the host: `cuda_stream` completes when the whole output is in host memory.  One staging
 * buffer per concurrently used stream.  Each (device, cuda_stream) pair gets its own pair of
 * copy streams, so calls issued on different streams overlap one op's device-to-host drain with
 * another's host-to-device feed; calls on the same stream run in issue order.
 */
TRIOT_API int triot_embed_host(void* dst, const int64_t* dst_shape, const void* src,
                               const int64_t* src_shape, int d, int dtype, unsigned flags,
                               void* staging, size_t staging_bytes, void* cuda_stream);

/* The expected value (Alg 11) of a PMF in HOST memory: p streamed through the staging
 * buffer in chunks of its leading axes ("copied to the GPU in chunks"), each chunk's
 * triot_expected_value_offset written to a row in staging, the rows summed in chunk order
 * (triot_sum_rows) and the d (+1 with_mass) doubles copied to the host array `out`.  offset
 * (host, d entries, NULL = zeros): p is the block of a larger PMF at that tuple, as in
 * triot_expected_value_offset.  The staging buffer (device, 256-byte aligned) also holds the
 * reduction workspace (cleared by the call itself); `cuda_stream` completes when `out` is
 * written.  Deterministic for a fixed staging size. */
TRIOT_API int triot_expected_value_host(double* out, const void* p, const int64_t* shape,
                                        const int64_t* offset, int d, int dtype, int with_mass,
                                        void* staging, size_t staging_bytes, void* cuda_stream);

/* c (host, dense in iter_shape, NULL = element-wise min) = a OP b, all host buffers. */
TRIOT_API int triot_apply_binary_host(void* c, const void* a, const int64_t* a_shape,
                                      const void* b, const int64_t* b_shape,
                                      const int64_t* iter_shape, int d, int dtype, int op,
                                      void* staging, size_t staging_bytes, void* cuda_stream);

/* ---- NEXT-1: tensor views -------------------------------------------
 *
 * A view is a window of a dense row-major base tensor: "a tensor slice starting at index tuple
 * (i_1, ..., i_d) can be constructed by using a bias: bias <- tuple_to_index((i_1, ..., i_d),
 * x.data_shape(), d).  Any valid accesses to the tensor slice ... x.flat[bias + flat_index]"
 * (P:605), flat_index taken with respect to the base shape.  Views let an op work on "the
 * intersecting support" of PMFs with different origins without copying.  Every op on a
 * view behaves exactly as on a materialised copy of its window (the index tuple t is relative
 * to the window's start).
 */
typedef struct {
  void* data;                 /* device pointer to the BASE tensor's element 0                */
  const int64_t* base_shape;  /* the base tensor's d extents (dense, row-major)               */
  const int64_t* start;       /* first tuple of the window in the base; NULL = the origin      */
  const int64_t* shape;       /* the window's d extents; start[k] + shape[k] <= base_shape[k] */
} triot_view;

/* triot_embed on views: the dst window receives the src window, zero-padded (flags as
 * triot_embed).  Elements of the dst base outside the dst window are never written.  The
 * windows' address ranges must not overlap (checked conservatively on the spanned bytes). */
TRIOT_API int triot_embed_view(const triot_view* dst, const triot_view* src, int d, int dtype,
                               unsigned flags, void* cuda_stream);

/* triot_apply_binary on views: for t in iter_shape (NULL = min of the a and b windows),
 * c_view[t] = a_view[t] OP b_view[t]; c's window must contain iter_shape.  In-place is allowed
 * only for the identical view (c == a or c == b) with iter_shape equal to its window. */
TRIOT_API int triot_apply_binary_view(const triot_view* c, const triot_view* a,
                                      const triot_view* b, const int64_t* iter_shape, int d,
                                      int dtype, int op, void* cuda_stream);

/* triot_expected_value on a view (Alg 11 over the window, t relative to the window's start):
 * out[k] = sum_t t_k p_view[t] for k < d, and out[d] = sum_t p_view[t] when with_mass != 0 (out
 * holds d or d + 1 doubles, device, 8-byte aligned, outside the view's base buffer).  Workspace
 * as triot_expected_value (triot_expected_value_workspace_size of the window's shape).  Same
 * numerics and determinism as the dense call; a window equal to its base gives the dense
 * call's value up to summation order. */
TRIOT_API int triot_expected_value_view(double* out, const triot_view* p, int d, int dtype,
                                        int with_mass, void* workspace, size_t workspace_bytes,
                                        void* cuda_stream);

/* ---- NEXT-2 / NEXT-3: the paper's Benchmarks 2 and 3 ----------------------------- */

/* Workspace bytes triot_inner_product needs (zero-filled once; the call leaves it ready). */
TRIOT_API int triot_inner_product_workspace_size(size_t* bytes);

/*
 * triot_inner_product -- Benchmark 2: "an inner product between two tensors ... (visiting only
 * tuple indices shared by both)", i.e. Alg 8's dot_product:
 *   *out = sum over t in prod[0, iter_shape[k]) of a[t] * b[t]
 * with a and b each indexed by its own shape; iter_shape NULL = element-wise min of the shapes.
 * fp64 accumulation (f32 inputs are widened), deterministic run to run.
 *   out: device pointer to one double.  workspace: see triot_inner_product_workspace_size.
 */
TRIOT_API int triot_inner_product(double* out, const void* a, const int64_t* a_shape,
                                  const void* b, const int64_t* b_shape,
                                  const int64_t* iter_shape, int d, int dtype, void* workspace,
                                  size_t workspace_bytes, void* cuda_stream);

/*
 * triot_fused_update -- Benchmark 3: "x[t] <- x[t] + y[t] * x[t] - z[t] is performed for all
 * tuples t that are valid with respect to the shape of x", in place on x (the
 * aliasing-safe apply_tensors idiom of P:601).  Evaluated as (x + (y * x)) - z with one IEEE
 * round-to-nearest rounding per operation.  y and z must contain x's shape and not overlap x.
 */
TRIOT_API int triot_fused_update(void* x, const int64_t* x_shape, const void* y,
                                 const int64_t* y_shape, const void* z, const int64_t* z_shape,
                                 int d, int dtype, void* cuda_stream);

/* ---- NEXT-4: naive multidimensional convolution (Alg 15; Benchmark 4) -------- */

/*
 * triot_naive_convolve -- result (dense, shape lhs_shape + rhs_shape - 1, written entirely) =
 * the convolution of Alg 15: for every lhs tuple t_l and rhs tuple t_r,
 *   result[t_l + t_r] += lhs[t_l] * rhs[t_r]        (result starts at 0.0)
 * "small problems are often much faster to solve using the naive approach".  Each
 * output is the sum of its rounded products in the order Alg 15 visits them (lexicographic in
 * t_l), so the result is bit-identical to the sequential algorithm.  All extents must be >= 1
 * and every tensor must have < 2^31 elements.  result must not overlap lhs or rhs.
 */
TRIOT_API int triot_naive_convolve(void* result, const void* lhs, const int64_t* lhs_shape,
                                   const void* rhs, const int64_t* rhs_shape, int d, int dtype,
                                   void* cuda_stream);

/* ---- diagnostics (host only; no device work, usable without a GPU) ---------------------- */

/*
 * triot_plan_describe -- writes, as one JSON object into buf (NUL-terminated, truncated to
 * buf_len), the launch plan the library would use for an op on these shapes: canonical axes
 * (unit axes dropped, contiguous axes merged), vector width, per-digit extents, the
 * per-step carry increment, per-tensor strides/carry deltas, and the fast-division magics.
 *   op: 0 = embed (shapes[0]=dst, shapes[1]=src, flags as triot_embed),
 *       1 = binary (shapes[0]=c or NULL, shapes[1]=a, shapes[2]=b, iter or NULL; `flags`
 *           carries the triot_binop),
 *       2 = expected value (shapes[0]=p),
 *       3 = inner product (shapes[0]=a, shapes[1]=b, iter or NULL),
 *       4 = fused update (shapes[0]=x, shapes[1]=y, shapes[2]=z),
 *       5 = naive convolution (shapes[0]=lhs, shapes[1]=rhs).
 *   ptr_mod32: byte offsets modulo 32 of each tensor's data pointer (alignment model).
 *   mode, warps: the work decomposition to describe (0 = contiguous chunk per warp, 1 = grid
 *              stride, over `warps` warps; 2 = contiguous chunk per block of the expected-value
 *              bulk-copy kernel, over `warps` blocks); the real call picks them from the SM count.
 * Returns a triot_status (validation errors exactly as the real call would report them).
 */
TRIOT_API int triot_plan_describe(int op, const int64_t* const* shapes, const int64_t* iter_shape,
                                  int d, int dtype, unsigned flags, const unsigned* ptr_mod32,
                                  int mode, uint64_t warps, char* buf, size_t buf_len);

/*
 * triot_set_launch_policy -- tuning hook (thread-local): force the work decomposition of this
 * thread's subsequent calls.  mode: -1 = automatic (default), 0 = contiguous chunk per warp,
 * 1 = grid stride, 2 / 3 = the expected value's bulk-copy (cp.async.bulk + mbarrier) pipeline
 * with 32 KB / 16 KB stages (other ops treat 2 and 3 as automatic), 4 = chunk per warp with the
 * expected value's block partials summed by a second kernel instead of the last block (other
 * ops treat 4 as 0), 5 = automatic without row windows (short odd rows and misaligned outputs
 * take flat vectors / element accesses instead; A/B measurements); blocks_per_sm: 0 = the
 * default for the mode.  Results are bit-identical under every
 * policy for embed and binary; the expected value's summation order follows the policy (it
 * stays deterministic for a fixed policy).  Used by tools/tune.py; not needed otherwise.
 */
TRIOT_API int triot_set_launch_policy(int mode, int blocks_per_sm);

/* The Granlund-Montgomery round-up magic the kernels use to divide by an invariant extent
 * (P:143 notes that division is slow; it is done once per thread with a multiply-high):
 *   q = (umulhi(n, mul) + ((n - umulhi(n, mul)) >> (shift & 0xff))) >> (shift >> 8)
 * equals n / divisor for every 32-bit n.  divisor must be >= 1. */
TRIOT_API int triot_fastdiv_magic(uint32_t divisor, uint32_t* mul, uint32_t* shift);


#ifdef __cplusplus
}
#endif

#endif /* TRIOT_H_ */
