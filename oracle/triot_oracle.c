/*
 * triot_oracle.c -- the CPU oracle for the TRIOT hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the CUDA library under
 * paper_1608_00099_b200/ and its Python binding) may include, link, load or call this file.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs use
 * it.  It shares no code, header, table or constant generator with the CUDA path.
 *
 * What it is: a plain, slow, single-threaded, obviously-correct transcription of the paper's
 * definitions, in the paper's order and notation.  Citation keys: P:n = line n of the paper
 * text (arxiv 1608.00099, "TRIOT: Faster tensor manipulation in C++11"); DESIGN.md lists every
 * reading taken where the paper is silent.
 *
 *   - tuple_to_index           Alg 2, verbatim; the Horner form of the P:50 sum.
 *   - advance_tuple            Alg 3, verbatim; lexicographic odometer.
 *   - index_to_tuple           the %-and-/ derivation of P:139.
 *   - reindex                  Alg 4, verbatim.
 *   - reindex_powers_of_2      Alg 12, verbatim.
 *   - embed                    Alg 9 apply_tensors with the Benchmark-1 body
 *                              "xV = yV", iterated over dst's shape, zero outside
 *                              src (zero padding).
 *   - apply_binary             Alg 9 apply_tensors with body c = a OP b, each operand indexed
 *                              by its own shape.
 *   - expected_value           Alg 11 with one tensor: m_k = sum_t t_k * p[t].
 *   - expected_value_abs       sum_t |t_k * p[t]|: the scale of the signed-input tolerance
 *                               over Alg 11's terms.
 *
 * Every loop is the paper's: t starts at the zero tuple (Alg 6's memset), every tensor
 * offset is recomputed from the full tuple with Alg 2 (never the "offset is just i" shortcut of
 * P:101), and t advances with Alg 3, N = prod(counter) times (the bound of Alg 13).
 *
 * Build: gcc -O2 -fno-fast-math -ffp-contract=off -fPIC -shared (never -Ofast: the paper's
 * flag would turn on FTZ/DAZ and FMA contraction and break bit parity).
 *
 * Parity pins: tests/test_oracle_pins.py checks every function here against values the paper
 * prints (651), closed forms, numpy library special cases and brute force;
 * expected_value_abs by exact-rational brute force on signed inputs and the closed form
 * p == -1 -> N (n_k - 1) / 2 (test_ev_abs_scale_*).  No function in this file is "parity
 * unpinned".
 */
#include <stdint.h>
#include <string.h>

typedef uint64_t u64;

/* element types and binary ops; the numeric values mirror the public C-ABI enums, but this file
 * does not include that header (the oracle shares no header with the CUDA path). */
enum { OR_F32 = 0, OR_F64 = 1 };
enum { OR_ADD = 0, OR_SUB = 1, OR_MUL = 2, OR_DIV = 3 };

/* ------------------------------------------------------------------------------------------
 * L0: scalar index arithmetic
 * ---------------------------------------------------------------------------------------- */

/* Alg 2: tuple to flat index with respect to shape (Horner's rule). */
u64 oracle_tuple_to_index(const u64* tup, const u64* shape, unsigned int dimension) {
  u64 res = 0;
  unsigned int k;
  for (k = 0; k < dimension - 1; ++k) {
    res += tup[k];
    res *= shape[k + 1];
  }
  res += tup[k];
  return res;
}

/* Alg 3: advance tup to its next lexicographic value with respect to shape. */
void oracle_advance_tuple(u64* tup, const u64* shape, unsigned int dimension) {
  ++tup[dimension - 1];
  for (unsigned int k = dimension - 1; k >= 1; --k)
    if (tup[k] >= shape[k]) {
      /* Perform carry operation: */
      ++tup[k - 1];
      tup[k] = 0;
    } else
      /* No more carry operations: */
      return;
}

/* t_{d-1} = x_index % s_{d-1}; subtract it, divide by s_{d-1}, repeat. */
void oracle_index_to_tuple(u64 index, const u64* shape, unsigned int dimension, u64* tup) {
  for (int i = (int)dimension - 1; i >= 0; --i) {
    tup[i] = index % shape[i];
    index = (index - tup[i]) / shape[i];
  }
}

/* Alg 4: reindex a flat index from shape to new_shape. */
u64 oracle_reindex(u64 index, const u64* shape, const u64* new_shape, unsigned int dimension) {
  u64 new_index = 0;
  u64 new_axis_product_from_right = 1;
  for (int i = (int)dimension - 1; index > 0 && i >= 0; --i) {
    u64 next_axis = shape[i];
    u64 new_next_axis = new_shape[i];
    u64 next_value = index % next_axis;
    new_index += next_value * new_axis_product_from_right;
    index /= next_axis;
    new_axis_product_from_right *= new_next_axis;
  }
  return new_index;
}

/* Alg 12: Alg 4 for power-of-two axes, with mask and shift. */
u64 oracle_reindex_powers_of_2(u64 index, const unsigned int* log_shape,
                               const unsigned int* new_log_shape, unsigned int dimension) {
  u64 new_index = 0;
  unsigned int new_axis_sum_from_right = 0;
  for (int i = (int)dimension - 1; index > 0 && i >= 0; --i) {
    u64 next_log_axis = log_shape[i];
    u64 new_next_log_axis = new_log_shape[i];
    u64 next_value = index & ((1ul << next_log_axis) - 1);
    new_index += (next_value << new_axis_sum_from_right);
    index >>= next_log_axis;
    new_axis_sum_from_right += (unsigned int)new_next_log_axis;
  }
  return new_index;
}

static u64 flat_size(const u64* shape, unsigned int dimension) {
  u64 n = 1;
  for (unsigned int k = 0; k < dimension; ++k) n *= shape[k];
  return n;
}

/* Enumerate every tuple of shape with Alg 3 starting from the zero tuple, writing the tuples
 * row by row into out (N x dimension).  Used by the tests to check bijection, order and the
 * per-digit carry counts of the P:129 amortisation argument. */
void oracle_enumerate(const u64* shape, unsigned int dimension, u64* out) {
  u64 t[64];
  u64 n = flat_size(shape, dimension);
  memset(t, 0, sizeof(t));
  for (u64 i = 0; i < n; ++i) {
    memcpy(out + i * dimension, t, dimension * sizeof(u64));
    oracle_advance_tuple(t, shape, dimension);
  }
}

/* ------------------------------------------------------------------------------------------
 * L4: the three hot-path operations
 * ---------------------------------------------------------------------------------------- */

/* Zero-padded embed, the apply_tensors body "xV = yV" of P:508-513 iterated over
 * dst's shape: dst[t] = src[t] if t_k < src_shape[k] for every k, else +0.0 (all-zero bits).
 * Elements are moved as raw bytes (esz = 4 or 8), so NaN payloads, -0.0 and subnormals survive.
 * region_only != 0: iterate over min(dst_shape, src_shape) only and leave the rest of dst as is. */
void oracle_embed(void* dst, const u64* dst_shape, const void* src, const u64* src_shape,
                  unsigned int dimension, unsigned int esz, int region_only) {
  u64 counter_shape[64];
  u64 t[64];
  unsigned char* d = (unsigned char*)dst;
  const unsigned char* s = (const unsigned char*)src;
  for (unsigned int k = 0; k < dimension; ++k)
    counter_shape[k] = region_only ? (dst_shape[k] < src_shape[k] ? dst_shape[k] : src_shape[k])
                                   : dst_shape[k];
  u64 n = flat_size(counter_shape, dimension);
  memset(t, 0, sizeof(t));
  for (u64 i = 0; i < n; ++i) {
    u64 dst_index = oracle_tuple_to_index(t, dst_shape, dimension);
    int in_bounds = 1;
    for (unsigned int k = 0; k < dimension; ++k)
      if (!(t[k] < src_shape[k])) in_bounds = 0;
    if (in_bounds) {
      u64 src_index = oracle_tuple_to_index(t, src_shape, dimension);
      memcpy(d + dst_index * esz, s + src_index * esz, esz);
    } else {
      memset(d + dst_index * esz, 0, esz);
    }
    oracle_advance_tuple(t, counter_shape, dimension);
  }
}

static double op_f64(double a, double b, int op) {
  switch (op) {
    case OR_ADD: return a + b;
    case OR_SUB: return a - b;
    case OR_MUL: return a * b;
    default: return a / b;
  }
}

static float op_f32(float a, float b, int op) {
  switch (op) {
    case OR_ADD: return a + b;
    case OR_SUB: return a - b;
    case OR_MUL: return a * b;
    default: return a / b;
  }
}

/* Element-wise binary op over tensors of different shapes (Alg 9 apply_tensors, P:320-326;
 * "the product of two or more probability mass functions with varying support"):
 * for every t in iter_shape, c[t] = a[t] OP b[t], each operand indexed by its own shape. */
void oracle_apply_binary(void* c, const u64* c_shape, const void* a, const u64* a_shape,
                         const void* b, const u64* b_shape, const u64* iter_shape,
                         unsigned int dimension, int dtype, int op) {
  u64 t[64];
  u64 n = flat_size(iter_shape, dimension);
  memset(t, 0, sizeof(t));
  for (u64 i = 0; i < n; ++i) {
    u64 ci = oracle_tuple_to_index(t, c_shape, dimension);
    u64 ai = oracle_tuple_to_index(t, a_shape, dimension);
    u64 bi = oracle_tuple_to_index(t, b_shape, dimension);
    if (dtype == OR_F64)
      ((double*)c)[ci] = op_f64(((const double*)a)[ai], ((const double*)b)[bi], op);
    else
      ((float*)c)[ci] = op_f32(((const float*)a)[ai], ((const float*)b)[bi], op);
    oracle_advance_tuple(t, iter_shape, dimension);
  }
}

/* Alg 11 with a single tensor: result[k] += counter[k] * xV for every tuple.
 * means[k] receives the Neumaier-compensated sum (the comparison target), plain[k] (if not NULL)
 * the literal sequential fp64 sum of Alg 11.  Each term is (double)t_k * (double)p[t], rounded
 * once.  No normalisation: Alg 11 never divides by sum(p). */
void oracle_expected_value(double* means, double* plain, const void* p, const u64* shape,
                           unsigned int dimension, int dtype) {
  u64 t[64];
  double sum[64], comp[64], lit[64];
  u64 n = flat_size(shape, dimension);
  memset(t, 0, sizeof(t));
  for (unsigned int k = 0; k < dimension; ++k) sum[k] = comp[k] = lit[k] = 0.0;
  for (u64 i = 0; i < n; ++i) {
    u64 pi = oracle_tuple_to_index(t, shape, dimension);
    double xV = dtype == OR_F64 ? ((const double*)p)[pi] : (double)((const float*)p)[pi];
    for (unsigned int k = 0; k < dimension; ++k) {
      double term = (double)t[k] * xV;
      lit[k] += term;
      /* Neumaier's improvement of Kahan summation */
      double s = sum[k] + term;
      if ((sum[k] >= 0 ? sum[k] : -sum[k]) >= (term >= 0 ? term : -term))
        comp[k] += (sum[k] - s) + term;
      else
        comp[k] += (term - s) + sum[k];
      sum[k] = s;
    }
    oracle_advance_tuple(t, shape, dimension);
  }
  for (unsigned int k = 0; k < dimension; ++k) {
    means[k] = sum[k] + comp[k];
    if (plain) plain[k] = lit[k];
  }
}

/* Sum of |t_k * p[t]| per axis: the scale of the 1e-12 relative bound for signed inputs. */
void oracle_expected_value_abs(double* out, const void* p, const u64* shape,
                               unsigned int dimension, int dtype) {
  u64 t[64];
  u64 n = flat_size(shape, dimension);
  memset(t, 0, sizeof(t));
  for (unsigned int k = 0; k < dimension; ++k) out[k] = 0.0;
  for (u64 i = 0; i < n; ++i) {
    u64 pi = oracle_tuple_to_index(t, shape, dimension);
    double xV = dtype == OR_F64 ? ((const double*)p)[pi] : (double)((const float*)p)[pi];
    for (unsigned int k = 0; k < dimension; ++k) {
      double term = (double)t[k] * xV;
      out[k] += term >= 0 ? term : -term;
    }
    oracle_advance_tuple(t, shape, dimension);
  }
}

/* ------------------------------------------------------------------------------------------
 * NEXT-1: tensor views ("a tensor slice starting at index tuple (i_1, ..., i_d) can
 * be constructed by using a bias: bias <- tuple_to_index((i_1, ..., i_d), x.data_shape(), d).
 * Any valid accesses to the tensor slice x_slice[flat_index] can be performed as
 * x.flat[bias + flat_index]"), where flat_index of a window tuple t is taken with respect to the
 * BASE shape (the window's elements are not contiguous in the base).  P:613: views window the
 * intersecting support of PMFs.  A view is (base, base_shape, start, window).
 * ---------------------------------------------------------------------------------------- */

/* the bias of a slice starting at tuple `start`. */
u64 oracle_view_bias(const u64* start, const u64* base_shape, unsigned int dimension) {
  return oracle_tuple_to_index(start, base_shape, dimension);
}

/* embed between views: iterate t over the dst window (or min(dst, src windows) if region_only),
 * dst_view[t] = (t < src window) ? src_view[t] : +0.0, with view[t] = base.flat[bias +
 * tuple_to_index(t, base_shape)]. */
void oracle_embed_view(void* dst, const u64* dst_base, const u64* dst_start, const u64* dst_win,
                       const void* src, const u64* src_base, const u64* src_start,
                       const u64* src_win, unsigned int dimension, unsigned int esz,
                       int region_only) {
  u64 counter_shape[64];
  u64 t[64];
  unsigned char* d = (unsigned char*)dst;
  const unsigned char* s = (const unsigned char*)src;
  u64 dst_bias = oracle_view_bias(dst_start, dst_base, dimension);
  u64 src_bias = oracle_view_bias(src_start, src_base, dimension);
  for (unsigned int k = 0; k < dimension; ++k)
    counter_shape[k] = region_only ? (dst_win[k] < src_win[k] ? dst_win[k] : src_win[k])
                                   : dst_win[k];
  u64 n = flat_size(counter_shape, dimension);
  memset(t, 0, sizeof(t));
  for (u64 i = 0; i < n; ++i) {
    u64 dst_index = dst_bias + oracle_tuple_to_index(t, dst_base, dimension);
    int in_bounds = 1;
    for (unsigned int k = 0; k < dimension; ++k)
      if (!(t[k] < src_win[k])) in_bounds = 0;
    if (in_bounds) {
      u64 src_index = src_bias + oracle_tuple_to_index(t, src_base, dimension);
      memcpy(d + dst_index * esz, s + src_index * esz, esz);
    } else {
      memset(d + dst_index * esz, 0, esz);
    }
    oracle_advance_tuple(t, counter_shape, dimension);
  }
}

/* binary op between views: for t in iter, c_view[t] = a_view[t] OP b_view[t]. */
void oracle_apply_binary_view(void* c, const u64* c_base, const u64* c_start, const void* a,
                              const u64* a_base, const u64* a_start, const void* b,
                              const u64* b_base, const u64* b_start, const u64* iter_shape,
                              unsigned int dimension, int dtype, int op) {
  u64 t[64];
  u64 n = flat_size(iter_shape, dimension);
  u64 cb = oracle_view_bias(c_start, c_base, dimension);
  u64 ab = oracle_view_bias(a_start, a_base, dimension);
  u64 bb = oracle_view_bias(b_start, b_base, dimension);
  memset(t, 0, sizeof(t));
  for (u64 i = 0; i < n; ++i) {
    u64 ci = cb + oracle_tuple_to_index(t, c_base, dimension);
    u64 ai = ab + oracle_tuple_to_index(t, a_base, dimension);
    u64 bi = bb + oracle_tuple_to_index(t, b_base, dimension);
    if (dtype == OR_F64)
      ((double*)c)[ci] = op_f64(((const double*)a)[ai], ((const double*)b)[bi], op);
    else
      ((float*)c)[ci] = op_f32(((const float*)a)[ai], ((const float*)b)[bi], op);
    oracle_advance_tuple(t, iter_shape, dimension);
  }
}

/* ------------------------------------------------------------------------------------------
 * NEXT-2 / NEXT-3: the paper's Benchmarks 2 and 3
 * ---------------------------------------------------------------------------------------- */

/* Benchmark 2 / Alg 8 dot_product: tot += xV * yV over the tuples of iter_shape
 * ("visiting only tuple indices shared by both").  *out = Neumaier-compensated sum of the
 * fp64 products (each product rounded once), *plain = the literal sequential sum of Alg 8. */
void oracle_inner_product(double* out, double* plain, const void* a, const u64* a_shape,
                          const void* b, const u64* b_shape, const u64* iter_shape,
                          unsigned int dimension, int dtype) {
  u64 t[64];
  u64 n = flat_size(iter_shape, dimension);
  double sum = 0.0, comp = 0.0, tot = 0.0;
  memset(t, 0, sizeof(t));
  for (u64 i = 0; i < n; ++i) {
    u64 ai = oracle_tuple_to_index(t, a_shape, dimension);
    u64 bi = oracle_tuple_to_index(t, b_shape, dimension);
    double xV = dtype == OR_F64 ? ((const double*)a)[ai] : (double)((const float*)a)[ai];
    double yV = dtype == OR_F64 ? ((const double*)b)[bi] : (double)((const float*)b)[bi];
    double term = xV * yV;
    tot += term;
    double s = sum + term;
    if ((sum >= 0 ? sum : -sum) >= (term >= 0 ? term : -term))
      comp += (sum - s) + term;
    else
      comp += (term - s) + sum;
    sum = s;
    oracle_advance_tuple(t, iter_shape, dimension);
  }
  *out = sum + comp;
  if (plain) *plain = tot;
}

/* Benchmark 3: "x[t] <- x[t] + y[t] * x[t] - z[t] is performed for all tuples t that are
 * valid with respect to the shape of x", written as apply_tensors with x by reference (the
 * aliasing-safe idiom of P:601).  C evaluation order, one rounding per operation:
 * (x + (y * x)) - z. */
void oracle_fused_update(void* x, const u64* x_shape, const void* y, const u64* y_shape,
                         const void* z, const u64* z_shape, unsigned int dimension, int dtype) {
  u64 t[64];
  u64 n = flat_size(x_shape, dimension);
  memset(t, 0, sizeof(t));
  for (u64 i = 0; i < n; ++i) {
    u64 xi = oracle_tuple_to_index(t, x_shape, dimension);
    u64 yi = oracle_tuple_to_index(t, y_shape, dimension);
    u64 zi = oracle_tuple_to_index(t, z_shape, dimension);
    if (dtype == OR_F64) {
      double* xv = (double*)x;
      xv[xi] = xv[xi] + ((const double*)y)[yi] * xv[xi] - ((const double*)z)[zi];
    } else {
      float* xv = (float*)x;
      xv[xi] = xv[xi] + ((const float*)y)[yi] * xv[xi] - ((const float*)z)[zi];
    }
    oracle_advance_tuple(t, x_shape, dimension);
  }
}

/* ------------------------------------------------------------------------------------------
 * NEXT-4: naive multidimensional convolution, Alg 15 (Benchmark 4)
 * ---------------------------------------------------------------------------------------- */

/* Alg 15: result has shape lhs + rhs - 1, is filled with 0.0, then for every
 * lhs tuple (outer enumerate_for_each_tensors) and every rhs tuple (inner one):
 * counter_result = counter_lhs + counter_rhs;
 * result.flat()[tuple_to_index(counter_result, result.data_shape())] += lhs_val * rhs_val
 * -- one rounding for the product, one for the sum.  All extents must be >= 1. */
void oracle_naive_convolve(void* result, const void* lhs, const u64* lhs_shape, const void* rhs,
                           const u64* rhs_shape, unsigned int dimension, int dtype) {
  u64 res_shape[64], tl[64], tr[64], tres[64];
  for (unsigned int k = 0; k < dimension; ++k) res_shape[k] = lhs_shape[k] + rhs_shape[k] - 1;
  u64 nres = flat_size(res_shape, dimension);
  u64 nl = flat_size(lhs_shape, dimension), nr = flat_size(rhs_shape, dimension);
  if (dtype == OR_F64)
    for (u64 i = 0; i < nres; ++i) ((double*)result)[i] = 0.0;
  else
    for (u64 i = 0; i < nres; ++i) ((float*)result)[i] = 0.0f;
  memset(tl, 0, sizeof(tl));
  for (u64 i = 0; i < nl; ++i) {
    u64 li = oracle_tuple_to_index(tl, lhs_shape, dimension);
    memset(tr, 0, sizeof(tr));
    for (u64 j = 0; j < nr; ++j) {
      u64 ri = oracle_tuple_to_index(tr, rhs_shape, dimension);
      for (unsigned int k = 0; k < dimension; ++k) tres[k] = tl[k] + tr[k];
      u64 oi = oracle_tuple_to_index(tres, res_shape, dimension);
      if (dtype == OR_F64)
        ((double*)result)[oi] += ((const double*)lhs)[li] * ((const double*)rhs)[ri];
      else
        ((float*)result)[oi] += ((const float*)lhs)[li] * ((const float*)rhs)[ri];
      oracle_advance_tuple(tr, rhs_shape, dimension);
    }
    oracle_advance_tuple(tl, lhs_shape, dimension);
  }
}
