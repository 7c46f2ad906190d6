// plan.cpp -- validation, canonicalisation and descriptor geometry (host only).
// See plan.hpp for the mapping to the paper's Alg 6-9; DESIGN.md §Plan for the rules.
#include "plan.hpp"

#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <string>

#include "../../include/triot.h"

namespace triot {

// ------------------------------------------------------------------------------ errors

static thread_local char g_err[512] = {0};

int set_error(int status, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return status;
}
void clear_error() { g_err[0] = 0; }
const char* last_error() { return g_err; }

// ------------------------------------------------------------------------------ fast division

void fastdiv_magic(uint32_t div, uint32_t* mul, uint32_t* shift) {
  // l = ceil(log2 div); m = floor(2^32 (2^l - div) / div) + 1; s1 = min(l,1); s2 = max(l-1,0)
  uint32_t l = 0;
  while (l < 32 && (1ull << l) < div) ++l;
  uint64_t m = ((((1ull << l) - div) << 32) / div) + 1;
  uint32_t s1 = l < 1 ? l : 1;
  uint32_t s2 = l > 0 ? l - 1 : 0;
  *mul = (uint32_t)m;
  *shift = s1 | (s2 << 8);
}

// ------------------------------------------------------------------------------ helpers

static const uint64_t kMaxBytes = 1ull << 62;

// Checks extents of one shape; sets numel.  P:48 assumes s_i >= 1; zero extents are allowed
// (reading R15) and negative ones rejected.
static int check_shape(const char* name, const int64_t* s, int d, int esz, uint64_t* numel) {
  if (!s) return set_error(TRIOT_ERR_NULL_POINTER, "NullPointer: shape of '%s' is NULL", name);
  uint64_t n = 1;
  bool zero = false;
  for (int k = 0; k < d; ++k) {
    if (s[k] < 0)
      return set_error(TRIOT_ERR_BAD_SHAPE, "BadShape: tensor '%s' axis %d has extent %lld", name,
                       k, (long long)s[k]);
    if (s[k] == 0) zero = true;
  }
  if (zero) {
    *numel = 0;
    return TRIOT_OK;
  }
  for (int k = 0; k < d; ++k) {
    uint64_t e = (uint64_t)s[k];
    if (e != 0 && n > (kMaxBytes / (uint64_t)esz) / e)
      return set_error(TRIOT_ERR_BAD_SHAPE, "BadShape: tensor '%s' has >= 2^62 bytes", name);
    n *= e;
  }
  *numel = n;
  return TRIOT_OK;
}

static int check_ptr(const char* name, const void* p, uint64_t numel, int esz) {
  if (numel == 0) return TRIOT_OK;
  if (!p) return set_error(TRIOT_ERR_NULL_POINTER, "NullPointer: data of '%s' is NULL", name);
  if (((uintptr_t)p) % (uintptr_t)esz)
    return set_error(TRIOT_ERR_MISALIGNED,
                     "Misaligned: data of '%s' (%p) is not aligned to its %d-byte element", name,
                     p, esz);
  return TRIOT_OK;
}

static bool overlap(const void* a, uint64_t na, const void* b, uint64_t nb, int esz) {
  if (na == 0 || nb == 0) return false;
  uintptr_t a0 = (uintptr_t)a, a1 = a0 + na * (uint64_t)esz;
  uintptr_t b0 = (uintptr_t)b, b1 = b0 + nb * (uint64_t)esz;
  return a0 < b1 && b0 < a1;
}

static int dtype_size(int dtype) { return dtype == TRIOT_F32 ? 4 : dtype == TRIOT_F64 ? 8 : 0; }

// Horner strides of a shape (Alg 2 / P:50): sigma_k = prod_{j>k} s_j.
static void strides_of(const int64_t* s, int d, uint64_t* sig) {
  uint64_t acc = 1;
  for (int k = d - 1; k >= 0; --k) {
    sig[k] = acc;
    acc *= (uint64_t)s[k];
  }
}

// ------------------------------------------------------------------------------ core planner
//
// Input: counter extents n[0..d-1], per tensor Horner strides, embed bounds bnd (min(src, n)).
// Output: g's canonical axes, digits and per-tensor accessors.

struct Axis {
  uint64_t n, bnd;
  uint64_t sig[TRIOT_MAXT];
  int orig, merged;
};

static int ilog2(uint64_t v) {
  int l = 0;
  while ((1ull << l) < v) ++l;
  return l;
}

static void finish_geometry(Geom& g, int nt);

// Flat-vector geometry: digits are the canonical axes at element granularity; vector v covers
// counter elements [v*V, v*V + V) (the last one may be partial).  A tensor gets full-width
// access iff it is dense with the counter (its strides are the counter's Horner strides) and
// 32-B aligned.
static void plan_flat(Geom& g, const Axis* ax, int na, int nt, bool bounds, const uint64_t* n0) {
  // 32-byte vectors; the expected value takes 64-byte units (two 32-byte loads per lane) when a
  // row is longer than a unit, i.e. at most one wrap per unit: the per-unit digit bookkeeping
  // is then paid once per 64 bytes (ev_flat_kernel, VB = 64)
  const int V = (g.op == OP_EV && ax[na - 1].n > (uint64_t)(64 / g.esz) ? 64 : 32) / g.esz;
  g.flat = true;
  g.V = V;
  g.R = 1;
  g.collapsed = false;
  g.D = na;
  g.lgL = ilog2((uint64_t)V);
  uint64_t hs = 1;  // counter Horner stride, innermost first
  uint64_t cstr[TRIOT_MAXD];
  for (int k = na - 1; k >= 0; --k) {
    cstr[k] = hs;
    hs *= ax[k].n;
  }
  for (int k = 0; k < na; ++k) {
    g.ext[k] = ax[k].n;
    g.bnd[k] = bounds ? ax[k].bnd : ax[k].n;
    for (int x = 0; x < nt; ++x) g.t[x].sig[k] = ax[k].sig[x];
  }
  for (int x = 0; x < nt; ++x) {
    bool dense = ((uintptr_t)g.t[x].ptr % 32) == 0;
    for (int k = 0; k < na; ++k)
      if (ax[k].sig[x] != cstr[k]) dense = false;
    g.t[x].vec = dense;
    g.t[x].rho = 0;
    g.t[x].tau = ax[na - 1].sig[x];
  }
  g.rowmul = g.colmul = 0;
  g.srows = g.scols = 0;
  g.vfull = g.vany = 0;
  g.N = 1;
  for (int k = 0; k < na; ++k) g.N *= ax[k].n;
  g.nvec = (g.N + V - 1) / V;
  g.nsteps = (g.nvec + 31) / 32;
  finish_geometry(g, nt);
  for (int j = 0; j <= TRIOT_MAXD; ++j) g.slot_of_axis[j] = -1;
  for (int k = 0; k < na; ++k) g.slot_of_axis[ax[k].orig] = k;
  g.nslots = na;
  if (g.N == 1 && n0[ax[0].orig] == 1) g.slot_of_axis[ax[0].orig] = -1;
  g.slot_of_axis[g.d] = na + 1;  // the mass
}

// Dense expected value with a short odd innermost extent n (no vector width divides it): a
// vector is one row of n contiguous elements, the digits are the outer axes (D = na - 1), and
// ev_rows_kernel stages tiles of whole rows in shared memory with bulk copies -- each thread
// sums its rows from shared memory (mass + column moment by suffix sums, ~4 instructions per
// element instead of the flat kernel's per-element odometer).  Needs a 16-byte aligned p (the
// bulk copies) and 3 <= n <= kEvRowsMax.
static const uint64_t kEvRowsMax = 31;
static void plan_ev_rows(Geom& g, const Axis* ax, int na, const uint64_t* n0) {
  const uint64_t n = ax[na - 1].n;
  g.evrows = true;
  g.flat = g.rows = false;
  g.V = 1;
  g.R = 1;
  g.collapsed = false;
  g.lgL = 0;
  g.D = na - 1;
  for (int k = 0; k < na - 1; ++k) {
    g.ext[k] = ax[k].n;
    g.bnd[k] = ax[k].n;
    g.t[0].sig[k] = ax[k].sig[0];
  }
  g.rowlen = (uint32_t)n;
  g.Dc = na;
  for (int k = 0; k < na; ++k) {
    g.cn[k] = ax[k].n;
    g.corig[k] = ax[k].orig;
    g.cmerged[k] = ax[k].merged;
  }
  g.t[0].vec = false;
  g.t[0].rho = 0;
  g.t[0].tau = ax[na - 1].sig[0];
  g.rowmul = g.colmul = 0;
  g.srows = g.scols = 0;
  g.vfull = g.vany = 0;
  g.N = 1;
  for (int k = 0; k < na; ++k) g.N *= ax[k].n;
  g.nvec = g.N / n;  // rows
  g.nsteps = (g.nvec + 31) / 32;
  finish_geometry(g, 1);
  for (int j = 0; j <= TRIOT_MAXD; ++j) g.slot_of_axis[j] = -1;
  for (int k = 0; k < na - 1; ++k) g.slot_of_axis[ax[k].orig] = k;  // outer axes
  g.slot_of_axis[ax[na - 1].orig] = na - 1;                          // the column moment
  g.nslots = na;
  g.slot_of_axis[g.d] = na;                                          // the mass (slot D + 1)
  (void)n0;
}

// Row windows: the longest innermost extent taken by row windows, per op (measured on B200,
// embed rows of 33 stream faster as flat vectors, whose only gather is src;
// binary rows up to 63 stream 1.7x faster as row windows, flat vectors gather both operands).
// Thread-local switch so the tuning hook (triot_set_launch_policy mode 5) can turn them off.
static const uint64_t kRowsMaxEmbed = 31, kRowsMaxBinary = 64;
// Rows up to this length take row windows when the output is misaligned (one window per group;
// the kernel's multiply-high division stays exact while e * n < 2^32, e < 32 n + 256).
static const uint64_t kRowsMaxLong = 4096;
// Rows this long take a warp per row (no per-element table lookups).
static const uint64_t kRowsWarpMin = 128;
static thread_local bool g_rows_on = true;
void set_rows_enabled(bool on) { g_rows_on = on; }
bool rows_enabled() { return g_rows_on; }

// Row-window geometry: digits are the outer canonical axes (a single unit digit when there is
// none); a "vector" is one counter row of n = rowlen elements; every tensor keeps its row
// offset (Horner over the outer digits, Alg 2) and its innermost stride tau.  A tensor is
// "dense" (vec) iff its offset of counter element f is f itself, so the kernel addresses it
// from the window base without the row offset.
static void plan_rows(Geom& g, const Axis* ax, int na, int nt, bool bounds) {
  g.rows = true;
  g.flat = false;
  g.V = 1;
  g.R = 1;
  g.collapsed = false;
  g.lgL = 0;
  const Axis& in = ax[na - 1];
  const uint64_t n = in.n;
  g.rowlen = n;
  g.rmag = (1ull << 32) / n + 1;  // n >= 3: fits 32 bits; umulhi(e, rmag) == e / n (e n < 2^32)
  // windows per group: >= 16 elements per lane, at most 8 and at most 248 / n (the group's
  // element indices stay below 2^13 for the magic; rows over 248 take one window, e < 32 n + 256,
  // where e * n < 2^32 keeps it exact up to kRowsMaxLong).  Measured on B200 against fixed 1, 2, 4, 8
  // windows per group (DESIGN.md §7 row windows): within 1-5 % of the best fixed choice.
  g.rwin = (16 + n - 1) / n;
  if (g.rwin > 8) g.rwin = 8;
  if (g.rwin > 248 / n) g.rwin = 248 / n;
  if (g.rwin < 1) g.rwin = 1;
  uint64_t cstr[TRIOT_MAXD];
  uint64_t hs = 1;
  for (int k = na - 1; k >= 0; --k) {
    cstr[k] = hs;
    hs *= ax[k].n;
  }
  if (na == 1) {  // one row: a single unit digit
    g.D = 1;
    g.ext[0] = 1;
    g.bnd[0] = 1;
    for (int x = 0; x < nt; ++x) g.t[x].sig[0] = 0;
  } else {
    g.D = na - 1;
    for (int k = 0; k < na - 1; ++k) {
      g.ext[k] = ax[k].n;
      g.bnd[k] = bounds ? ax[k].bnd : ax[k].n;
      for (int x = 0; x < nt; ++x) g.t[x].sig[k] = ax[k].sig[x];
    }
  }
  for (int x = 0; x < nt; ++x) {
    bool dense = in.sig[x] == 1;
    for (int k = 0; k < na; ++k)
      if (ax[k].sig[x] != cstr[k]) dense = false;
    g.t[x].vec = dense;
    g.t[x].rho = 0;
    g.t[x].tau = in.sig[x];
  }
  // long rows into an output not dense in the counter (a view window, a region, a wide c): a
  // warp per row saves the table lookup of the output offset (B200: embed into a (512)^3 view
  // at (63,63,63) 3.35 -> 4.61 TB/s); dense outputs keep the table (C2 with dst off by 4 B:
  // 4.72 table vs 4.44 warp per row; f64 rows of 128: 5.72 vs 5.08)
  g.rwarp = n >= kRowsWarpMin && !g.t[0].vec && g.op != OP_EV;
  g.rowmul = g.colmul = 0;
  g.srows = 1;
  g.scols = g.all_oob ? 0 : (bounds ? in.bnd : n);
  g.vfull = g.vany = 0;
  g.N = 1;
  for (int k = 0; k < na; ++k) g.N *= ax[k].n;
  g.nvec = g.N / n;
  g.nsteps = (g.nvec + 31) / 32;
  finish_geometry(g, nt);
  for (int j = 0; j <= TRIOT_MAXD; ++j) g.slot_of_axis[j] = -1;
  g.nslots = 0;
}

static void build(Geom& g, const uint64_t* n, const uint64_t (*sig)[TRIOT_MAXD],
                  const uint64_t* bnd, bool allow_merge, bool bounds) {
  const int d = g.d, nt = g.ntensor;
  // 1. drop unit axes ("if some axes have trivial length 1, then those axes can simply
  //    be ignored"); keep at least one axis.
  Axis ax[TRIOT_MAXD];
  int na = 0;
  for (int k = 0; k < d; ++k) {
    if (n[k] == 1) continue;
    Axis a;
    a.n = n[k];
    a.bnd = bnd ? bnd[k] : n[k];
    for (int x = 0; x < nt; ++x) a.sig[x] = sig[x][k];
    a.orig = k;
    a.merged = 1;
    ax[na++] = a;
  }
  if (na == 0) {
    Axis a;
    a.n = 1;
    a.bnd = 1;
    for (int x = 0; x < nt; ++x) a.sig[x] = sig[x][d - 1];
    a.orig = d - 1;
    a.merged = 1;
    ax[na++] = a;
  }
  // 2. merge adjacent axes whose strides compose in every tensor (and, for embed, whose inner
  //    axis is never out of bounds), so that merged offsets are still Horner sums.
  if (allow_merge) {
    int j = na - 1;
    while (j > 0) {
      Axis& o = ax[j - 1];
      Axis& i = ax[j];
      bool ok = true;
      for (int x = 0; x < nt; ++x)
        if (o.sig[x] != i.n * i.sig[x]) ok = false;
      if (bounds && i.bnd != i.n) ok = false;
      if (ok) {
        Axis m;
        m.n = o.n * i.n;
        m.bnd = o.bnd * i.n;
        for (int x = 0; x < nt; ++x) m.sig[x] = i.sig[x];
        m.orig = i.orig;
        m.merged = o.merged + i.merged;
        ax[j - 1] = m;
        for (int q = j; q + 1 < na; ++q) ax[q] = ax[q + 1];
        --na;
        --j;  // the merged axis sits at j-1: next try (j-2, j-1)
      } else {
        --j;
      }
    }
  }
  g.Dc = na;
  for (int k = 0; k < na; ++k) {
    g.cn[k] = ax[k].n;
    g.corig[k] = ax[k].orig;
    g.cmerged[k] = ax[k].merged;
  }

  // 3. vector geometry: V in {32 B, 16 B, 1 element}; case (a) V | n_last, case (b) rows
  //    shorter than a vector, R = V / n_last whole rows per vector.
  const int vmax = 32 / g.esz;
  const int cands[3] = {vmax, 16 / g.esz, 1};
  int best = -1;
  long best_score = -1;
  struct Cand {
    int V, R, D;
    bool collapsed;
    bool vec[TRIOT_MAXT];
  } cc[3];
  const uint64_t nl = ax[na - 1].n;
  for (int ci = 0; ci < 3; ++ci) {
    int V = cands[ci];
    Cand c;
    c.V = V;
    c.R = 1;
    c.collapsed = false;
    if (nl % (uint64_t)V == 0) {
      c.D = na;
    } else if (na >= 2 && nl < (uint64_t)V && (uint64_t)V % nl == 0 &&
               ax[na - 2].n % ((uint64_t)V / nl) == 0) {
      c.R = V / (int)nl;
      c.collapsed = true;
      c.D = na - 1;
    } else {
      cc[ci].V = 0;
      continue;
    }
    // per-tensor wide-access legality: contiguous inside the vector and V*esz aligned
    int nvec_ok = 0;
    for (int x = 0; x < nt; ++x) {
      bool ok = V > 1;
      uint64_t tau = ax[na - 1].sig[x];
      if (tau != 1) ok = false;
      if (c.collapsed && ax[na - 2].sig[x] != nl) ok = false;
      if ((uintptr_t)g.t[x].ptr % (uintptr_t)(V * g.esz)) ok = false;
      for (int k = 0; k < na - (c.collapsed ? 2 : 1); ++k)
        if (ax[k].sig[x] % (uint64_t)V) ok = false;
      if (c.collapsed && (ax[na - 2].sig[x] * (uint64_t)c.R) % (uint64_t)V) ok = false;
      c.vec[x] = ok;
      nvec_ok += ok ? 1 : 0;
    }
    cc[ci] = c;
    long score = (c.vec[0] ? 1000 : 0) + nvec_ok * 100 + V;
    if (score > best_score) {
      best_score = score;
      best = ci;
    }
  }
  // flat vectors: when no vector width fits the innermost extent (odd extents: 3, 5, 7, 999),
  // take V consecutive elements of the flattened counter instead of one element per lane, for
  // the ops that have flat kernels.  The counter-dense tensors then still get full-width access.
  // Flat vectors store 32 B at a time only into an output dense in the counter and 32-B
  // aligned; any other output (a view window, a misaligned base) takes row windows up to
  // kRowsMaxLong, whose lane-consecutive element stores coalesce at any alignment.
  bool shift_build = false;
  bool out_flat_vec = ((uintptr_t)g.t[0].ptr % 32) == 0;
  {
    uint64_t hs = 1;
    for (int k = na - 1; k >= 0; --k) {
      if (ax[k].sig[0] != hs) out_flat_vec = false;
      hs *= ax[k].n;
    }
  }
  uint64_t rows_max = !g_rows_on ? 0 : g.op == OP_EMBED ? kRowsMaxEmbed : kRowsMaxBinary;
  if (g_rows_on && !out_flat_vec) rows_max = kRowsMaxLong;
  if (cc[best].V == 1 && vmax > 1 && g.rows_ok && nl >= 3 && nl <= rows_max) {
    plan_rows(g, ax, na, nt, bounds);
    return;
  }
  // The output (dst / c) cannot take wide stores although a vector width fits its rows -- its
  // base is only element-aligned (a view at an odd offset, a sliced buffer): element stores at a
  // 32-byte lane stride write partial sectors (C2 with dst offset by 4 B: 1.4 TB/s), so rows up
  // to kRowsMaxLong take row windows, whose lane-consecutive accesses coalesce at any alignment;
  // longer rows (a fully merged copy) are cut into segments of a divisor L <= kRowsMaxLong.
  // An embed / binary op whose output is dense in the counter and only misaligned (a slice of a
  // buffer) keeps the 32-byte vectors and stores them shifted to the 32-byte grid
  // (embed_shift_kernel, binary_shift_kernel).
  if ((g.op == OP_EMBED || g.op == OP_BINARY) && g_rows_on && cc[0].V == vmax &&
      !cc[0].vec[0]) {
    const uintptr_t mis = (uintptr_t)g.t[0].ptr % 32;
    bool dense0 = mis % (uintptr_t)g.esz == 0;
    uint64_t hs = 1;
    for (int k = na - 1; k >= 0; --k) {
      if (ax[k].sig[0] != hs) dense0 = false;
      hs *= ax[k].n;
    }
    if (dense0 && mis != 0) {  // the 32-byte candidate, whatever the others scored
      g.dshift = (uint32_t)(mis / (uintptr_t)g.esz);
      shift_build = true;
      best = 0;
    }
  }
  const bool long_ok = g.rows_ok && g_rows_on && g.op != OP_EV && nl >= 3 && !shift_build;
  if ((cc[best].V > 1 && !cc[best].vec[0] && long_ok) ||
      (cc[best].V == 1 && vmax > 1 && !out_flat_vec && long_ok)) {
    // rows over 512 elements are cut into segments of a divisor L in [64, 512] when one
    // exists: a warp step is 32 rows, so rows of thousands of elements leave too few warps
    // (a merged 84 M-element copy in rows of 4,096: 640 warps, 1.3 TB/s)
    uint64_t L = 0;
    if (nl > 512)
      for (uint64_t c = 512; c >= 64 && !L; --c)
        if (nl % c == 0) L = c;
    if (!L && nl <= kRowsMaxLong) {
      plan_rows(g, ax, na, nt, bounds);
      return;
    }
    if (L && na < TRIOT_MAXD) {
      // split the innermost axis into (nl / L segments, L): a row is one segment; the embed
      // bound m of the unsplit axis becomes a per-segment column bound (kernel: segm)
      Axis sx[TRIOT_MAXD + 1];
      for (int k = 0; k < na - 1; ++k) sx[k] = ax[k];
      Axis seg = ax[na - 1], in = ax[na - 1];
      seg.n = nl / L;
      seg.bnd = seg.n;
      for (int x = 0; x < nt; ++x) seg.sig[x] = ax[na - 1].sig[x] * L;
      in.n = L;
      in.bnd = L;
      sx[na - 1] = seg;
      sx[na] = in;
      plan_rows(g, sx, na + 1, nt, bounds);
      g.seglen = L;
      g.segm = bounds ? ax[na - 1].bnd : nl;
      return;
    }
  }
  // ... and a dense p whose rows would only take 16-byte vectors (n = 12, 20, 28 floats; 6, 10,
  // 14 ... doubles): half-width loads stream at 3.7-4.4 TB/s, the row tiles at 5.2-5.7 and, past
  // their 31 elements, the 64-byte flat units at 5.0-5.7 (268 MB, profiles/r02_ev_narrow*.jsonl)
  const bool narrow = g.op == OP_EV && !g.view && g_rows_on && cc[best].V > 1 &&
                      cc[best].V * g.esz < 32 && !cc[best].collapsed;
  if (narrow && g.flat_ok && nl > kEvRowsMax && nl > (uint64_t)(64 / g.esz) &&
      ((uintptr_t)g.t[0].ptr % 32) == 0) {
    plan_flat(g, ax, na, nt, bounds, n);
    return;
  }
  if ((cc[best].V == 1 || narrow) && vmax > 1 && g.op == OP_EV && !g.view && g_rows_on && na >= 2 &&
      nl >= 3 && nl <= kEvRowsMax && ((uintptr_t)g.t[0].ptr % 16) == 0) {
    plan_ev_rows(g, ax, na, n);
    return;
  }
  if (cc[best].V == 1 && vmax > 1 && g.flat_ok) {
    plan_flat(g, ax, na, nt, bounds, n);
    return;
  }
  // The expected value of a view window whose rows take no vector width (odd lengths): vectors
  // of V elements padded past the row end (the vector digit runs to ceil(n / V)); the kernel
  // loads element-wise and masks the padding (ev_view_kernel, evpad) -- instead of one element
  // per lane and odometer step.
  const bool evpad = g.op == OP_EV && g.view && g_rows_on && cc[best].V == 1 && vmax > 1 &&
                     nl > (uint64_t)vmax;
  if (evpad) {
    Cand p;
    p.V = vmax;
    p.R = 1;
    p.collapsed = false;
    p.D = na;
    for (int x = 0; x < nt; ++x) p.vec[x] = false;
    cc[0] = p;
    best = 0;
  }
  const Cand& c = cc[best];
  g.V = c.V;
  g.R = c.R;
  g.collapsed = c.collapsed;
  g.D = c.D;
  const int D = g.D;
  const uint64_t V = (uint64_t)c.V;
  // digit k < D-1 is canonical axis k; the vector digit D-1 is axis na-1 (a) or na-2 (b)
  for (int k = 0; k < D - 1; ++k) {
    g.ext[k] = ax[k].n;
    g.bnd[k] = ax[k].bnd;
    for (int x = 0; x < nt; ++x) g.t[x].sig[k] = ax[k].sig[x];
  }
  if (!c.collapsed) {
    const Axis& a = ax[na - 1];
    g.ext[D - 1] = a.n / V;
    g.bnd[D - 1] = g.ext[D - 1];
    for (int x = 0; x < nt; ++x) {
      g.t[x].sig[D - 1] = V * a.sig[x];
      g.t[x].rho = 0;
      g.t[x].tau = a.sig[x];
    }
    g.lgL = ilog2(V);
    g.rowmul = 0;
    g.colmul = V;
    g.srows = 1;
    g.scols = bounds ? a.bnd : a.n;
    g.vfull = g.scols / V;
    g.vany = (g.scols + V - 1) / V;
  } else {
    const Axis& r = ax[na - 2];
    const Axis& a = ax[na - 1];
    const uint64_t R = (uint64_t)c.R;
    g.ext[D - 1] = r.n / R;
    g.bnd[D - 1] = g.ext[D - 1];
    for (int x = 0; x < nt; ++x) {
      g.t[x].sig[D - 1] = R * r.sig[x];
      g.t[x].rho = r.sig[x];
      g.t[x].tau = a.sig[x];
    }
    g.lgL = ilog2(a.n);
    g.rowmul = R;
    g.colmul = 0;
    g.srows = bounds ? r.bnd : r.n;
    g.scols = bounds ? a.bnd : a.n;
    g.vfull = g.scols >= a.n ? g.srows / R : 0;
    g.vany = g.scols > 0 ? (g.srows + R - 1) / R : 0;
  }
  if (!bounds) {
    g.vfull = g.vany = g.ext[D - 1];
    for (int k = 0; k < D; ++k) g.bnd[k] = g.ext[k];
  }
  if (g.all_oob) {
    g.vfull = g.vany = 0;
  }
  for (int x = 0; x < nt; ++x) g.t[x].vec = c.vec[x];

  // 4. totals, the +32-vector step in mixed radix, carry deltas, fast-division magics
  g.N = 1;
  for (int k = 0; k < na; ++k) g.N *= ax[k].n;
  g.nvec = g.N / V;
  if (evpad) {
    g.ext[D - 1] = (nl + V - 1) / V;
    g.bnd[D - 1] = g.ext[D - 1];
    g.scols = nl;  // elements of a row; the padding past it is masked
    g.evpad = true;
    g.nvec = g.N / nl * g.ext[D - 1];
  }
  g.nsteps = (g.nvec + 31) / 32;
  finish_geometry(g, nt);
  // 6. expected-value weight slots: digit k<D-1 -> axis; vector digit -> last (a) or row axis (b)
  for (int j = 0; j <= TRIOT_MAXD; ++j) g.slot_of_axis[j] = -1;
  for (int k = 0; k < D - 1; ++k) g.slot_of_axis[ax[k].orig] = k;
  if (!c.collapsed) {
    g.slot_of_axis[ax[na - 1].orig] = D - 1;
    g.nslots = D;
  } else {
    g.slot_of_axis[ax[na - 2].orig] = D - 1;
    g.slot_of_axis[ax[na - 1].orig] = D;
    g.nslots = D + 1;
  }
  if (g.N == 1 && n[ax[0].orig] == 1) g.slot_of_axis[ax[0].orig] = -1;  // weight 0 anyway
  g.slot_of_axis[d] = D + 1;  // the total mass (read only when requested)
}

// carry deltas, the default decomposition, fast-division magics, index width
static void finish_geometry(Geom& g, int nt) {
  const int D = g.D;
  const uint64_t V = (uint64_t)g.V;
  for (int x = 0; x < nt; ++x) {
    g.t[x].kap[0] = 0;
    for (int k = 1; k < D; ++k) g.t[x].kap[k] = g.t[x].sig[k - 1] - g.ext[k] * g.t[x].sig[k];
  }
  set_decomposition(g, 0, 1);
  for (int k = 0; k < D; ++k) {
    uint32_t e = g.ext[k] >= 1 && g.ext[k] <= 0xffffffffull ? (uint32_t)g.ext[k] : 1;
    fastdiv_magic(e, &g.fdm[k], &g.fds[k]);
  }
  // decode by shifts when every digit extent the decode divides by is a power of two
  g.pow2 = true;
  for (int k = 1; k < D; ++k) {
    const uint64_t e = g.ext[k];
    if (e == 0 || (e & (e - 1)) != 0) g.pow2 = false;
    g.lg[k] = (uint8_t)ilog2(e);
  }
  // tensor 0 dense in the digit space: its offset of digit vector v is v * (last digit stride)
  g.lin0 = g.t[0].sig[D - 1];
  for (int k = 0; k + 1 < D; ++k)
    if (g.t[0].sig[k] != g.t[0].sig[k + 1] * g.ext[k + 1]) g.lin0 = 0;
  // 5. index width: 32-bit iff every offset, count and vector index fits, with room for the
  //    largest per-batch advance (K steps of up to 2^20 vectors)
  uint64_t mx = g.N + (1ull << 24) * V;
  for (int x = 0; x < nt; ++x)
    if (g.t[x].numel > mx) mx = g.t[x].numel;
  for (int k = 0; k < D; ++k)
    if (g.ext[k] + 32 > mx) mx = g.ext[k] + 32;
  g.idx64 = mx >= (1ull << 32) - 64;
}

void set_decomposition(Geom& g, int mode, uint64_t warps) {
  if (warps < 1) warps = 1;
  if (mode == 2) {
    // block chunks for the EV bulk-copy kernel: `warps` counts blocks here; each block owns a
    // multiple of SVEC vectors and its threads step by one block (TRIOT_BLOCK vectors)
    g.mode = 2;
    uint64_t per = (g.nvec + warps - 1) / warps;
    g.wmul = g.wspan = per;
    g.dv = TRIOT_EV_TMA_BLOCK;
  } else if (mode == 1) {
    g.mode = 1;
    g.wmul = 32;
    g.wspan = g.nvec;
    g.dv = 32 * warps;
  } else {
    g.mode = 0;
    uint64_t q = (g.nsteps + warps - 1) / warps;
    if (q < 1) q = 1;
    g.wmul = g.wspan = 32 * q;
    g.dv = 32;
  }
  set_step(g);
}

// the step of dv vectors in mixed radix (digit 0 absorbs the rest; it only matters past the
// end).  Flat vectors: the kernel walks the vector's V elements with +1 steps, then skips
// (dv-1)*V.
void set_step(Geom& g) {
  const int D = g.D;
  uint64_t rem = g.flat ? (g.dv - 1) * (uint64_t)g.V : g.dv;
  for (int k = D - 1; k >= 1; --k) {
    g.dlt[k] = rem % g.ext[k];
    rem /= g.ext[k];
  }
  g.dlt[0] = rem;
  g.khi = -1;
  g.klo = D;
  for (int k = 0; k < D; ++k)
    if (g.dlt[k]) {
      if (k > g.khi) g.khi = k;
      if (k < g.klo) g.klo = k;
    }
  if (g.khi < 0) {  // a zero step (flat vectors with dv == 1): no digit changes
    g.khi = -1;
    g.klo = D;
  }
  for (int x = 0; x < g.ntensor; ++x) {
    uint64_t st = 0;
    for (int k = 0; k < D; ++k) st += g.dlt[k] * g.t[x].sig[k];
    g.t[x].step = st;
  }
  // embed zero runs: a step of exactly one unit of digit khi < D-1 and dst offsets linear in it
  g.zmask = 0;
  if (g.op == OP_EMBED && !g.flat && !g.rows && g.mode == 0 && g.dv == 32 && g.khi >= 0 && g.khi < D - 1 &&
      g.dlt[g.khi] == 1 && g.t[0].vec && g.V * g.esz == 32) {
    bool ok = true;
    for (int k = 0; k < D; ++k) ok = ok && (k == g.khi ? true : g.dlt[k] == 0);
    for (int k = 1; k <= g.khi; ++k) ok = ok && g.t[0].kap[k] == 0;
    if (ok) {
      g.zmask = (uint32_t)((2ull << g.khi) - 1ull);
      uint64_t nsub = 1;
      for (int k = g.khi; k >= 0; --k) {
        nsub *= g.ext[k];
        g.zn[k] = nsub;
        if (nsub < (1ull << 32)) fastdiv_magic((uint32_t)nsub, &g.zdm[k], &g.zds[k]);
      }
    }
  }
}

// ------------------------------------------------------------------------------ public planners

// A tensor argument: a window of `shape` extents whose element t sits at ptr + Horner(t, base)
// elements -- a dense tensor (window == base, start 0) or a view (bias =
// tuple_to_index(start, base_shape); element t of the slice is base.flat[bias + Horner(t, base)]).
struct TArg {
  const char* name;
  const void* ptr;             // the window's element 0 (base + bias)
  int64_t shape[TRIOT_MAXD];   // window extents
  uint64_t sig[TRIOT_MAXD];    // Horner strides of the base shape
  uint64_t numel;              // window elements
  uint64_t span;               // elements from ptr through the window's last element (0 if empty)
  const void* base;            // the base buffer (== ptr for a dense tensor)
  int64_t start[TRIOT_MAXD];   // the window's start tuple in the base (0 for a dense tensor)
  int d;
};

static void targ_span(TArg& t, int d) {
  if (t.numel == 0) {
    t.span = 0;
    return;
  }
  uint64_t last = 0;
  for (int k = 0; k < d; ++k) last += (uint64_t)(t.shape[k] - 1) * t.sig[k];
  t.span = last + 1;
}

static int targ_dense(TArg& t, const char* name, const void* ptr, const int64_t* shape, int d,
                      int esz) {
  int st;
  t.name = name;
  if ((st = check_shape(name, shape, d, esz, &t.numel))) return st;
  for (int k = 0; k < d; ++k) t.shape[k] = shape[k];
  strides_of(shape, d, t.sig);
  t.ptr = ptr;
  t.base = ptr;
  t.d = d;
  for (int k = 0; k < d; ++k) t.start[k] = 0;
  targ_span(t, d);
  return TRIOT_OK;
}

static int targ_view(TArg& t, const char* name, const triot_view* v, int d, int esz) {
  int st;
  t.name = name;
  if (!v) return set_error(TRIOT_ERR_NULL_POINTER, "NullPointer: view '%s' is NULL", name);
  uint64_t nbase;
  if ((st = check_shape(name, v->base_shape, d, esz, &nbase))) return st;
  if ((st = check_shape(name, v->shape, d, esz, &t.numel))) return st;
  strides_of(v->base_shape, d, t.sig);
  uint64_t bias = 0;
  for (int k = 0; k < d; ++k) {
    const int64_t s0 = v->start ? v->start[k] : 0;
    // shape and base_shape are >= 0 (check_shape), so the difference cannot overflow
    if (s0 < 0 || s0 > v->base_shape[k] - v->shape[k])
      return set_error(TRIOT_ERR_AXIS_OUT_OF_BOUNDS,
                       "AxisOutOfBounds: view '%s' axis %d: start %lld + window %lld > base "
                       "extent %lld",
                       name, k, (long long)s0, (long long)v->shape[k],
                       (long long)v->base_shape[k]);
    t.shape[k] = v->shape[k];
    t.start[k] = s0;
    bias += (uint64_t)s0 * t.sig[k];  // Horner of the start tuple
  }
  if ((st = check_ptr(name, v->data, t.numel, esz))) return st;
  // a non-empty window has s0_k <= base_k - 1 on every axis, so bias <= nbase - 1 and
  // bias * esz < 2^62 (check_shape); an empty window touches no memory and keeps bias 0 (its
  // base may have zero extents, where the strides were never bounded)
  if (t.numel == 0) bias = 0;
  t.ptr = (const char*)v->data + bias * (uint64_t)esz;
  t.base = v->data;
  t.d = d;
  targ_span(t, d);
  return TRIOT_OK;
}

// Two windows of one base laid out with the same strides share an element iff their boxes
// [start, start + shape) intersect on every axis (a base tuple has one address: digits k >= 1
// stay below their base extents); otherwise fall back to the conservative byte-span test.
static bool targ_overlap(const TArg& a, const TArg& b, int esz) {
  if (a.numel == 0 || b.numel == 0) return false;
  bool same_layout = a.base == b.base && a.d == b.d;
  for (int k = 0; same_layout && k < a.d; ++k) same_layout = a.sig[k] == b.sig[k];
  if (same_layout) {
    for (int k = 0; k < a.d; ++k)
      if (a.start[k] >= b.start[k] + b.shape[k] || b.start[k] >= a.start[k] + a.shape[k])
        return false;
    return true;
  }
  return overlap(a.ptr, a.span, b.ptr, b.span, esz);
}

static bool targ_same(const TArg& a, const TArg& b, int d) {
  if (a.ptr != b.ptr) return false;
  for (int k = 0; k < d; ++k)
    if (a.shape[k] != b.shape[k] || a.sig[k] != b.sig[k]) return false;
  return true;
}

static int check_common(int d, int dtype, int* esz) {
  if (d < 1 || d > TRIOT_MAXD)
    return set_error(TRIOT_ERR_UNSUPPORTED_DIMENSION,
                     "UnsupportedDimension: d = %d, supported 1..%d", d, TRIOT_MAXD);
  *esz = dtype_size(dtype);
  if (!*esz) return set_error(TRIOT_ERR_BAD_DTYPE_OR_OP, "BadDtype: dtype = %d", dtype);
  return TRIOT_OK;
}

static int plan_embed_core(Geom& g, const TArg& dst, const TArg& src, int d, int dtype, int esz,
                           unsigned flags) {
  bool region = (flags & TRIOT_EMBED_REGION_ONLY) != 0;
  uint64_t n[TRIOT_MAXD], bnd[TRIOT_MAXD];
  uint64_t N = 1;
  for (int k = 0; k < d; ++k) {
    uint64_t D_ = (uint64_t)dst.shape[k], S = (uint64_t)src.shape[k];
    n[k] = region ? (D_ < S ? D_ : S) : D_;
    bnd[k] = S < n[k] ? S : n[k];
    N *= n[k];
  }
  int st;
  if ((st = check_ptr("dst", dst.ptr, dst.numel, esz))) return st;
  // src is read only where t < src_shape inside the counter
  bool reads_src = N > 0 && src.numel > 0;
  if ((st = check_ptr("src", src.ptr, reads_src ? src.numel : 0, esz))) return st;
  if (reads_src && targ_overlap(dst, src, esz))
    return set_error(TRIOT_ERR_ALIASING, "Aliasing: dst and src overlap");
  g.op = OP_EMBED;
  g.flat_ok = true;
  g.rows_ok = true;
  g.esz = esz;
  g.dtype = dtype;
  g.flags = flags;
  g.d = d;
  g.ntensor = 2;
  g.t[0].ptr = dst.ptr;
  g.t[0].numel = dst.span;
  g.t[1].ptr = src.ptr;
  g.t[1].numel = src.span;
  if (N == 0) {
    g.empty = true;
    clear_error();
    return TRIOT_OK;
  }
  g.all_oob = src.numel == 0;
  uint64_t sig[TRIOT_MAXT][TRIOT_MAXD];
  for (int k = 0; k < d; ++k) {
    sig[0][k] = dst.sig[k];
    sig[1][k] = src.numel == 0 ? 0 : src.sig[k];
  }
  build(g, n, sig, bnd, /*allow_merge=*/true, /*bounds=*/!region);
  clear_error();
  return TRIOT_OK;
}

int plan_embed(Geom& g, void* dst, const int64_t* dst_shape, const void* src,
               const int64_t* src_shape, int d, int dtype, unsigned flags) {
  g = Geom();
  int esz, st;
  if ((st = check_common(d, dtype, &esz))) return st;
  if (flags & ~1u) return set_error(TRIOT_ERR_BAD_DTYPE_OR_OP, "BadFlags: flags = %u", flags);
  TArg td, ts;
  if ((st = targ_dense(td, "dst", dst, dst_shape, d, esz))) return st;
  if ((st = targ_dense(ts, "src", src, src_shape, d, esz))) return st;
  if ((st = check_ptr("dst", dst, td.numel, esz))) return st;
  return plan_embed_core(g, td, ts, d, dtype, esz, flags);
}

int plan_embed_view(Geom& g, const triot_view* dst, const triot_view* src, int d, int dtype,
                    unsigned flags) {
  g = Geom();
  int esz, st;
  if ((st = check_common(d, dtype, &esz))) return st;
  if (flags & ~1u) return set_error(TRIOT_ERR_BAD_DTYPE_OR_OP, "BadFlags: flags = %u", flags);
  TArg td, ts;
  if ((st = targ_view(td, "dst", dst, d, esz))) return st;
  if ((st = targ_view(ts, "src", src, d, esz))) return st;
  return plan_embed_core(g, td, ts, d, dtype, esz, flags);
}

static int plan_binary_core(Geom& g, const TArg& c, const TArg& a, const TArg& b,
                            const int64_t* it, int d, int dtype, int esz, int op) {
  uint64_t ni = 1;
  for (int k = 0; k < d; ++k) ni *= (uint64_t)it[k];
  // check_tensor_pack_bounds: the iteration shape must lie inside every operand
  const TArg* ts[3] = {&c, &a, &b};
  for (int x = 0; x < 3; ++x)
    for (int k = 0; k < d; ++k)
      if (it[k] > ts[x]->shape[k])
        return set_error(TRIOT_ERR_AXIS_OUT_OF_BOUNDS,
                         "AxisOutOfBounds: tensor '%s' axis %d: iteration extent %lld > tensor "
                         "extent %lld",
                         ts[x]->name, k, (long long)it[k], (long long)ts[x]->shape[k]);
  int st;
  if ((st = check_ptr("c", c.ptr, c.numel, esz))) return st;
  if (ni) {
    for (int x = 1; x < 3; ++x)
      if ((st = check_ptr(ts[x]->name, ts[x]->ptr, ts[x]->numel, esz))) return st;
    for (int x = 1; x < 3; ++x) {
      if (!targ_overlap(c, *ts[x], esz)) continue;
      bool inplace = targ_same(c, *ts[x], d);
      for (int k = 0; k < d && inplace; ++k)
        if (it[k] != c.shape[k]) inplace = false;
      if (!inplace)
        return set_error(TRIOT_ERR_ALIASING,
                         "Aliasing: c overlaps '%s' (only exact in-place c == %s with equal "
                         "shapes and iteration shape is allowed)",
                         ts[x]->name, ts[x]->name);
    }
  }
  g.op = OP_BINARY;
  g.flat_ok = true;
  g.rows_ok = true;
  g.esz = esz;
  g.dtype = dtype;
  g.binop = op;
  g.d = d;
  g.ntensor = 3;
  for (int x = 0; x < 3; ++x) {
    g.t[x].ptr = ts[x]->ptr;
    g.t[x].numel = ts[x]->span;
  }
  if (ni == 0) {
    g.empty = true;
    clear_error();
    return TRIOT_OK;
  }
  uint64_t n[TRIOT_MAXD];
  for (int k = 0; k < d; ++k) n[k] = (uint64_t)it[k];
  uint64_t sig[TRIOT_MAXT][TRIOT_MAXD];
  for (int x = 0; x < 3; ++x)
    for (int k = 0; k < d; ++k) sig[x][k] = ts[x]->sig[k];
  build(g, n, sig, nullptr, /*allow_merge=*/true, /*bounds=*/false);
  clear_error();
  return TRIOT_OK;
}

static int check_binop(int op) {
  if (op < TRIOT_ADD || op > TRIOT_DIV)
    return set_error(TRIOT_ERR_BAD_DTYPE_OR_OP, "BadOp: op = %d", op);
  return TRIOT_OK;
}

int plan_binary(Geom& g, void* c, const int64_t* c_shape, const void* a, const int64_t* a_shape,
                const void* b, const int64_t* b_shape, const int64_t* iter_shape, int d,
                int dtype, int op) {
  g = Geom();
  int esz, st;
  if ((st = check_common(d, dtype, &esz))) return st;
  if ((st = check_binop(op))) return st;
  TArg ta, tb, tc;
  if ((st = targ_dense(ta, "a", a, a_shape, d, esz))) return st;
  if ((st = targ_dense(tb, "b", b, b_shape, d, esz))) return st;
  int64_t it[TRIOT_MAXD];
  if (iter_shape) {
    uint64_t ni;
    if ((st = check_shape("iter", iter_shape, d, esz, &ni))) return st;
    for (int k = 0; k < d; ++k) it[k] = iter_shape[k];
  } else {
    for (int k = 0; k < d; ++k) it[k] = a_shape[k] < b_shape[k] ? a_shape[k] : b_shape[k];
  }
  if ((st = targ_dense(tc, "c", c, c_shape ? c_shape : it, d, esz))) return st;
  uint64_t ni = 1;
  for (int k = 0; k < d; ++k) ni *= (uint64_t)it[k];
  // element alignment of every operand that is touched
  if ((st = check_ptr("c", c, tc.numel, esz))) return st;
  if ((st = check_ptr("a", a, ni ? ta.numel : 0, esz))) return st;
  if ((st = check_ptr("b", b, ni ? tb.numel : 0, esz))) return st;
  return plan_binary_core(g, tc, ta, tb, it, d, dtype, esz, op);
}

int plan_binary_view(Geom& g, const triot_view* c, const triot_view* a, const triot_view* b,
                     const int64_t* iter_shape, int d, int dtype, int op) {
  g = Geom();
  int esz, st;
  if ((st = check_common(d, dtype, &esz))) return st;
  if ((st = check_binop(op))) return st;
  TArg ta, tb, tc;
  if ((st = targ_view(ta, "a", a, d, esz))) return st;
  if ((st = targ_view(tb, "b", b, d, esz))) return st;
  if ((st = targ_view(tc, "c", c, d, esz))) return st;
  int64_t it[TRIOT_MAXD];
  if (iter_shape) {
    uint64_t ni;
    if ((st = check_shape("iter", iter_shape, d, esz, &ni))) return st;
    for (int k = 0; k < d; ++k) it[k] = iter_shape[k];
  } else {
    for (int k = 0; k < d; ++k) it[k] = ta.shape[k] < tb.shape[k] ? ta.shape[k] : tb.shape[k];
  }
  return plan_binary_core(g, tc, ta, tb, it, d, dtype, esz, op);
}

// NEXT-2: Benchmark 2 / Alg 8 dot_product over iter (NULL = the shared tuples).
int plan_dot(Geom& g, const void* a, const int64_t* a_shape, const void* b,
             const int64_t* b_shape, const int64_t* iter_shape, int d, int dtype) {
  g = Geom();
  int esz, st;
  if ((st = check_common(d, dtype, &esz))) return st;
  TArg ta, tb;
  if ((st = targ_dense(ta, "a", a, a_shape, d, esz))) return st;
  if ((st = targ_dense(tb, "b", b, b_shape, d, esz))) return st;
  int64_t it[TRIOT_MAXD];
  if (iter_shape) {
    uint64_t ni;
    if ((st = check_shape("iter", iter_shape, d, esz, &ni))) return st;
    for (int k = 0; k < d; ++k) it[k] = iter_shape[k];
  } else {
    for (int k = 0; k < d; ++k) it[k] = a_shape[k] < b_shape[k] ? a_shape[k] : b_shape[k];
  }
  const TArg* ts[2] = {&ta, &tb};
  uint64_t ni = 1;
  for (int k = 0; k < d; ++k) ni *= (uint64_t)it[k];
  for (int x = 0; x < 2; ++x) {
    for (int k = 0; k < d; ++k)
      if (it[k] > ts[x]->shape[k])
        return set_error(TRIOT_ERR_AXIS_OUT_OF_BOUNDS,
                         "AxisOutOfBounds: tensor '%s' axis %d: iteration extent %lld > tensor "
                         "extent %lld",
                         ts[x]->name, k, (long long)it[k], (long long)ts[x]->shape[k]);
    if ((st = check_ptr(ts[x]->name, ts[x]->ptr, ni ? ts[x]->numel : 0, esz))) return st;
  }
  g.op = OP_DOT;
  g.esz = esz;
  g.dtype = dtype;
  g.d = d;
  g.nout = 1;
  g.ntensor = 2;
  for (int x = 0; x < 2; ++x) {
    g.t[x].ptr = ts[x]->ptr;
    g.t[x].numel = ts[x]->span;
  }
  if (ni == 0) {
    g.empty = true;
    clear_error();
    return TRIOT_OK;
  }
  uint64_t n[TRIOT_MAXD];
  uint64_t sig[TRIOT_MAXT][TRIOT_MAXD];
  for (int k = 0; k < d; ++k) {
    n[k] = (uint64_t)it[k];
    sig[0][k] = ta.sig[k];
    sig[1][k] = tb.sig[k];
  }
  build(g, n, sig, nullptr, /*allow_merge=*/true, /*bounds=*/false);
  for (int j = 0; j <= TRIOT_MAXD; ++j) g.slot_of_axis[j] = -1;
  g.slot_of_axis[0] = 0;
  clear_error();
  return TRIOT_OK;
}

// NEXT-3: Benchmark 3: x[t] <- x[t] + y[t]*x[t] - z[t] for t in x's shape, in place.
int plan_update(Geom& g, void* x, const int64_t* x_shape, const void* y, const int64_t* y_shape,
                const void* z, const int64_t* z_shape, int d, int dtype) {
  g = Geom();
  int esz, st;
  if ((st = check_common(d, dtype, &esz))) return st;
  TArg tx, ty, tz;
  if ((st = targ_dense(tx, "x", x, x_shape, d, esz))) return st;
  if ((st = targ_dense(ty, "y", y, y_shape, d, esz))) return st;
  if ((st = targ_dense(tz, "z", z, z_shape, d, esz))) return st;
  const TArg* ts[3] = {&tx, &ty, &tz};
  for (int q = 1; q < 3; ++q)
    for (int k = 0; k < d; ++k)
      if (x_shape[k] > ts[q]->shape[k])
        return set_error(TRIOT_ERR_AXIS_OUT_OF_BOUNDS,
                         "AxisOutOfBounds: tensor '%s' axis %d: iteration extent %lld > tensor "
                         "extent %lld",
                         ts[q]->name, k, (long long)x_shape[k], (long long)ts[q]->shape[k]);
  for (int q = 0; q < 3; ++q)
    if ((st = check_ptr(ts[q]->name, ts[q]->ptr, tx.numel ? ts[q]->numel : 0, esz))) return st;
  if (tx.numel)
    for (int q = 1; q < 3; ++q)
      if (targ_overlap(tx, *ts[q], esz))
        return set_error(TRIOT_ERR_ALIASING, "Aliasing: x overlaps '%s'", ts[q]->name);
  g.op = OP_UPDATE;
  g.esz = esz;
  g.dtype = dtype;
  g.d = d;
  g.ntensor = 3;
  for (int q = 0; q < 3; ++q) {
    g.t[q].ptr = ts[q]->ptr;
    g.t[q].numel = ts[q]->span;
  }
  if (tx.numel == 0) {
    g.empty = true;
    clear_error();
    return TRIOT_OK;
  }
  uint64_t n[TRIOT_MAXD];
  uint64_t sig[TRIOT_MAXT][TRIOT_MAXD];
  for (int k = 0; k < d; ++k) {
    n[k] = (uint64_t)x_shape[k];
    for (int q = 0; q < 3; ++q) sig[q][k] = ts[q]->sig[k];
  }
  build(g, n, sig, nullptr, /*allow_merge=*/true, /*bounds=*/false);
  clear_error();
  return TRIOT_OK;
}

// NEXT-4: Alg 15 naive convolution.  The launch uses its own descriptor layout
// (conv_kernel): ext/fdm/fds = result shape, bnd = lhs extents, dlt = rhs extents.
int plan_conv(Geom& g, void* result, const void* lhs, const int64_t* lhs_shape, const void* rhs,
              const int64_t* rhs_shape, int d, int dtype) {
  g = Geom();
  int esz, st;
  if ((st = check_common(d, dtype, &esz))) return st;
  TArg tl, tr;
  if ((st = targ_dense(tl, "lhs", lhs, lhs_shape, d, esz))) return st;
  if ((st = targ_dense(tr, "rhs", rhs, rhs_shape, d, esz))) return st;
  int64_t rs[TRIOT_MAXD];
  for (int k = 0; k < d; ++k) {
    if (lhs_shape[k] < 1 || rhs_shape[k] < 1)
      return set_error(TRIOT_ERR_BAD_SHAPE,
                       "BadShape: convolution operands need extents >= 1 (axis %d)", k);
    rs[k] = lhs_shape[k] + rhs_shape[k] - 1;
  }
  TArg to;
  if ((st = targ_dense(to, "result", result, rs, d, esz))) return st;
  const uint64_t lim = 1ull << 31;
  if (to.numel >= lim || tl.numel >= lim || tr.numel >= lim)
    return set_error(TRIOT_ERR_BAD_SHAPE, "BadShape: convolution tensors must have < 2^31 elements");
  if ((st = check_ptr("result", result, to.numel, esz))) return st;
  if ((st = check_ptr("lhs", lhs, tl.numel, esz))) return st;
  if ((st = check_ptr("rhs", rhs, tr.numel, esz))) return st;
  if (targ_overlap(to, tl, esz) || targ_overlap(to, tr, esz))
    return set_error(TRIOT_ERR_ALIASING, "Aliasing: result overlaps an operand");
  g.op = OP_CONV;
  g.esz = esz;
  g.dtype = dtype;
  g.d = d;
  g.D = d;
  g.V = 1;
  g.ntensor = 3;
  g.nvec = to.numel;
  g.N = to.numel;
  for (int k = 0; k < d; ++k) {
    g.ext[k] = (uint64_t)rs[k];
    g.bnd[k] = (uint64_t)lhs_shape[k];
    g.dlt[k] = (uint64_t)rhs_shape[k];
    fastdiv_magic((uint32_t)rs[k], &g.fdm[k], &g.fds[k]);
    g.t[0].sig[k] = tl.sig[k];
    g.t[1].sig[k] = tr.sig[k];
    g.t[2].sig[k] = to.sig[k];
  }
  g.t[0].ptr = lhs;
  g.t[1].ptr = rhs;
  g.t[2].ptr = result;
  g.t[0].numel = tl.numel;
  g.t[1].numel = tr.numel;
  g.t[2].numel = to.numel;
  clear_error();
  return TRIOT_OK;
}

int plan_ev(Geom& g, const void* p, const int64_t* shape, int d, int dtype) {
  g = Geom();
  if (d < 1 || d > TRIOT_MAXD)
    return set_error(TRIOT_ERR_UNSUPPORTED_DIMENSION,
                     "UnsupportedDimension: d = %d, supported 1..%d", d, TRIOT_MAXD);
  int esz = dtype_size(dtype);
  if (!esz) return set_error(TRIOT_ERR_BAD_DTYPE_OR_OP, "BadDtype: dtype = %d", dtype);
  uint64_t np_;
  int st;
  if ((st = check_shape("p", shape, d, esz, &np_))) return st;
  if ((st = check_ptr("p", p, np_, esz))) return st;
  g.op = OP_EV;
  g.flat_ok = true;
  g.esz = esz;
  g.dtype = dtype;
  g.d = d;
  g.ntensor = 1;
  g.t[0].ptr = p;
  g.t[0].numel = np_;
  if (np_ == 0) {
    g.empty = true;
    clear_error();
    return TRIOT_OK;
  }
  uint64_t n[TRIOT_MAXD];
  for (int k = 0; k < d; ++k) n[k] = (uint64_t)shape[k];
  uint64_t sig[TRIOT_MAXT][TRIOT_MAXD];
  strides_of(shape, d, sig[0]);
  // every digit is a weight (Alg 11 reads counter[k]), so axes are never merged
  build(g, n, sig, nullptr, /*allow_merge=*/false, /*bounds=*/false);
  clear_error();
  return TRIOT_OK;
}

// NEXT-1 for the third op: Alg 11 over a view's window (element t of the window is
// base.flat[bias + Horner(t, base shape)]).  The counter is the window; p's offsets follow the
// base strides, so the kernels track them with the odometer instead of assuming p is dense.
// No flat vectors (their loads assume a dense p): odd innermost extents take 1-element vectors.
int plan_ev_view(Geom& g, const triot_view* p, int d, int dtype) {
  g = Geom();
  int esz, st;
  if ((st = check_common(d, dtype, &esz))) return st;
  TArg tp;
  if ((st = targ_view(tp, "p", p, d, esz))) return st;
  g.op = OP_EV;
  g.view = true;
  g.flat_ok = false;
  g.esz = esz;
  g.dtype = dtype;
  g.d = d;
  g.ntensor = 1;
  g.t[0].ptr = tp.ptr;
  g.t[0].numel = tp.span;  // the index width must cover the window's span in the base
  if (tp.numel == 0) {
    g.empty = true;
    clear_error();
    return TRIOT_OK;
  }
  uint64_t n[TRIOT_MAXD];
  for (int k = 0; k < d; ++k) n[k] = (uint64_t)tp.shape[k];
  uint64_t sig[TRIOT_MAXT][TRIOT_MAXD];
  for (int k = 0; k < d; ++k) sig[0][k] = tp.sig[k];
  build(g, n, sig, nullptr, /*allow_merge=*/false, /*bounds=*/false);
  clear_error();
  return TRIOT_OK;
}

// ------------------------------------------------------------------------------ describe

static void arr(std::string& s, const char* key, const uint64_t* v, int n) {
  s += "\"";
  s += key;
  s += "\":[";
  char b[32];
  for (int i = 0; i < n; ++i) {
    snprintf(b, sizeof(b), "%s%llu", i ? "," : "", (unsigned long long)v[i]);
    s += b;
  }
  s += "],";
}
static void arri(std::string& s, const char* key, const int* v, int n) {
  s += "\"";
  s += key;
  s += "\":[";
  char b[32];
  for (int i = 0; i < n; ++i) {
    snprintf(b, sizeof(b), "%s%d", i ? "," : "", v[i]);
    s += b;
  }
  s += "],";
}
static void arr32(std::string& s, const char* key, const uint32_t* v, int n) {
  uint64_t w[TRIOT_MAXD];
  for (int i = 0; i < n; ++i) w[i] = v[i];
  arr(s, key, w, n);
}

std::string describe(const Geom& g) {
  std::string s = "{";
  char b[1024];
  snprintf(b, sizeof(b),
           "\"op\":%d,\"esz\":%d,\"d\":%d,\"empty\":%s,\"idx64\":%s,\"all_oob\":%s,\"Dc\":%d,"
           "\"D\":%d,\"V\":%d,\"R\":%d,\"lgL\":%d,\"collapsed\":%s,\"flat\":%s,\"N\":%llu,\"nvec\":%llu,"
           "\"nsteps\":%llu,\"mode\":%d,\"wmul\":%llu,\"wspan\":%llu,\"dv\":%llu,\"khi\":%d,\"klo\":%d,\"rowmul\":%llu,\"colmul\":%llu,\"vfull\":%llu,"
           "\"vany\":%llu,\"srows\":%llu,\"scols\":%llu,\"nslots\":%d,\"zmask\":%u,"
           "\"rows\":%s,\"rowlen\":%llu,\"rmag\":%llu,\"rwin\":%llu,\"pow2\":%s,\"lin0\":%llu,"
           "\"seglen\":%llu,\"segm\":%llu,\"rwarp\":%s,\"dshift\":%u,\"evpad\":%s,"
           "\"evrows\":%s,",
           g.op, g.esz, g.d, g.empty ? "true" : "false", g.idx64 ? "true" : "false",
           g.all_oob ? "true" : "false", g.Dc, g.D, g.V, g.R, g.lgL,
           g.collapsed ? "true" : "false", g.flat ? "true" : "false", (unsigned long long)g.N, (unsigned long long)g.nvec,
           (unsigned long long)g.nsteps, g.mode, (unsigned long long)g.wmul,
           (unsigned long long)g.wspan, (unsigned long long)g.dv, g.khi, g.klo, (unsigned long long)g.rowmul,
           (unsigned long long)g.colmul, (unsigned long long)g.vfull, (unsigned long long)g.vany,
           (unsigned long long)g.srows, (unsigned long long)g.scols, g.nslots, g.zmask,
           g.rows ? "true" : "false", (unsigned long long)g.rowlen, (unsigned long long)g.rmag,
           (unsigned long long)g.rwin, g.pow2 ? "true" : "false", (unsigned long long)g.lin0,
           (unsigned long long)g.seglen, (unsigned long long)g.segm, g.rwarp ? "true" : "false",
           g.dshift, g.evpad ? "true" : "false", g.evrows ? "true" : "false");
  s += b;
  arr(s, "cn", g.cn, g.Dc);
  arri(s, "corig", g.corig, g.Dc);
  arri(s, "cmerged", g.cmerged, g.Dc);
  arr(s, "ext", g.ext, g.D);
  arr(s, "dlt", g.dlt, g.D);
  arr(s, "bnd", g.bnd, g.D);
  arr(s, "zn", g.zn, g.D);
  arr32(s, "fdm", g.fdm, g.D);
  arr32(s, "fds", g.fds, g.D);
  arri(s, "slot_of_axis", g.slot_of_axis, g.d + 1);
  s += "\"t\":[";
  for (int x = 0; x < g.ntensor; ++x) {
    s += x ? ",{" : "{";
    arr(s, "sig", g.t[x].sig, g.D);
    arr(s, "kap", g.t[x].kap, g.D);
    snprintf(b, sizeof(b), "\"step\":%llu,\"rho\":%llu,\"tau\":%llu,\"vec\":%s,\"numel\":%llu}",
             (unsigned long long)g.t[x].step, (unsigned long long)g.t[x].rho,
             (unsigned long long)g.t[x].tau, g.t[x].vec ? "true" : "false",
             (unsigned long long)g.t[x].numel);
    s += b;
  }
  s += "]}";
  return s;
}

}  // namespace triot
