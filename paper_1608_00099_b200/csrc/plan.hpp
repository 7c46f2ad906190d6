// plan.hpp -- host side of the boundary: validation, canonicalisation and the launch plan.
//
// Pure host C++ (no CUDA headers), so the whole plan can be inspected without a GPU through
// triot_plan_describe().  The paper's structure it replaces:
//   - check_tensor_pack_bounds (Alg 8/9): one check over shapes;
//   - LinearTemplateSearch (Alg 7): runtime d -> compile-time instance; here an O(1)
//     table lookup on the canonical digit count (dispatch.cu);
//   - ForEachFixedDimension (Alg 6): the per-tuple loop nest; here the descriptor that
//     lets each GPU lane run the odometer of Alg 3 on a compile-time number of digits.
#pragma once
#include <stddef.h>
#include <stdint.h>

#include <string>

#include "../../include/triot.h"
#include "desc.h"

namespace triot {

struct Geom {
  int op = 0, esz = 0, dtype = 0, binop = 0;
  unsigned flags = 0;
  int d = 0;          // caller's dimension
  int ntensor = 0;
  bool empty = false; // nothing to launch (empty counter); EV still writes zeros
  bool idx64 = false;
  bool all_oob = false;
  // canonical axes (after unit-axis drop and merge), for describe()
  int Dc = 0;
  uint64_t cn[TRIOT_MAXD] = {};
  int corig[TRIOT_MAXD] = {};      // original axis of each canonical axis (innermost of a merge)
  int cmerged[TRIOT_MAXD] = {};    // number of original axes merged into it
  // digits
  int D = 0, V = 1, R = 1, lgL = 0;
  bool collapsed = false;
  bool flat = false;   // flat vectors: V consecutive counter elements across rows (odd extents)
  bool flat_ok = false;  // the op has flat-vector kernels (embed, binary, expected value)
  bool rows = false;     // row windows: a vector is one counter row (short odd innermost)
  bool evrows = false;   // dense EV with a short odd innermost extent: rows staged in shared
                         // memory by bulk copies (ev_rows_kernel); digits = the outer axes
  bool rows_ok = false;  // the op has row-window kernels (embed, binary)
  uint64_t rowlen = 0, rmag = 0, rwin = 1;
  uint64_t seglen = 0, segm = 0;   // rows are segments of a split axis; segm = its embed bound
  bool rwarp = false;              // long rows: a warp per row instead of the row table
  uint32_t dshift = 0;             // embed: dst dense but misaligned by this many elements
  bool evpad = false;              // EV of a view: vectors padded past odd rows (scols = n)
  uint64_t N = 0;
  uint64_t ext[TRIOT_MAXD] = {}, dlt[TRIOT_MAXD] = {}, bnd[TRIOT_MAXD] = {};
  uint32_t fdm[TRIOT_MAXD] = {}, fds[TRIOT_MAXD] = {};
  bool pow2 = false;                // every digit extent 1..D-1 a power of two
  uint8_t lg[TRIOT_MAXD] = {};
  uint64_t lin0 = 0;                // tensor 0 dense in the digit space: offset = v * lin0
  uint64_t nvec = 0, nsteps = 0;
  uint64_t wmul = 32, wspan = 32, dv = 32;   // decomposition (set_decomposition)
  int mode = 0;                              // 0 = chunk, 1 = stride, 2 = block chunk
  int khi = 0, klo = 0;
  uint64_t rowmul = 0, colmul = 0, vfull = 0, vany = 0, srows = 0, scols = 0;
  int slot_of_axis[TRIOT_MAXD + 1] = {};
  int nslots = 0;
  bool with_mass = false;   // EV: also write sum(p) after the d means
  int nout = -1;            // reduction outputs if not d (+mass): the inner product writes 1
  bool split = false;       // reductions: partials summed by a second (PDL) kernel
  uint32_t cluster = 0;     // reductions: the grid is one cluster of this many blocks (launch_geometry)
  int nax = 0;              // EV of a block of a larger PMF: per-axis coordinate offsets
  double offd[TRIOT_MAXD] = {};
  bool view = false;        // EV of a view: p is strided (offsets tracked by the odometer)
  uint32_t zmask = 0;       // embed zero runs (desc.h)
  uint64_t zn[TRIOT_MAXD] = {};
  uint32_t zdm[TRIOT_MAXD] = {}, zds[TRIOT_MAXD] = {};
  struct T {
    uint64_t sig[TRIOT_MAXD] = {}, kap[TRIOT_MAXD] = {};
    uint64_t step = 0, rho = 0, tau = 1;
    bool vec = false;
    const void* ptr = nullptr;
    uint64_t numel = 0;
  } t[TRIOT_MAXT];
};

// Each returns a triot_status; on error the thread-local message is set.
int plan_embed(Geom& g, void* dst, const int64_t* dst_shape, const void* src,
               const int64_t* src_shape, int d, int dtype, unsigned flags);
int plan_binary(Geom& g, void* c, const int64_t* c_shape, const void* a, const int64_t* a_shape,
                const void* b, const int64_t* b_shape, const int64_t* iter_shape, int d,
                int dtype, int op);
int plan_ev(Geom& g, const void* p, const int64_t* shape, int d, int dtype);
// NEXT-2 / NEXT-3: Benchmark 2 inner product and Benchmark 3 fused update
int plan_dot(Geom& g, const void* a, const int64_t* a_shape, const void* b,
             const int64_t* b_shape, const int64_t* iter_shape, int d, int dtype);
int plan_update(Geom& g, void* x, const int64_t* x_shape, const void* y, const int64_t* y_shape,
                const void* z, const int64_t* z_shape, int d, int dtype);
// NEXT-4: Alg 15 naive convolution
int plan_conv(Geom& g, void* result, const void* lhs, const int64_t* lhs_shape, const void* rhs,
              const int64_t* rhs_shape, int d, int dtype);
// NEXT-1: the same ops on views
int plan_embed_view(Geom& g, const triot_view* dst, const triot_view* src, int d, int dtype,
                    unsigned flags);
int plan_ev_view(Geom& g, const triot_view* p, int d, int dtype);
int plan_binary_view(Geom& g, const triot_view* c, const triot_view* a, const triot_view* b,
                     const int64_t* iter_shape, int d, int dtype, int op);

// Work decomposition over `warps` warps: mode 0 = contiguous chunk per warp, 1 = grid stride,
// 2 = contiguous chunk per block (EV bulk-copy kernel; `warps` is then the number of blocks).
// Sets wmul/wspan/dv and the mixed-radix digits of the per-step advance (dlt, khi, klo, step).
void set_decomposition(Geom& g, int mode, uint64_t warps);
// Row windows on/off for this thread (tuning hook, triot_set_launch_policy mode 5).
void set_rows_enabled(bool on);
bool rows_enabled();
// (Re)compute the mixed-radix digits of the per-step advance for the current g.dv.
void set_step(Geom& g);

// Granlund-Montgomery round-up magic for an invariant 32-bit divisor (>= 1).
void fastdiv_magic(uint32_t div, uint32_t* mul, uint32_t* shift);

std::string describe(const Geom& g);

// thread-local error detail
int set_error(int status, const char* fmt, ...);
void clear_error();
const char* last_error();

template <typename IDX>
void fill_desc(const Geom& g, Desc<IDX>& d) {
  for (int k = 0; k <= TRIOT_MAXD; ++k) d.slot_of_axis[k] = g.slot_of_axis[k];
  for (int k = 0; k < TRIOT_MAXD; ++k) {
    d.ext[k] = (IDX)g.ext[k];
    d.dlt[k] = (IDX)g.dlt[k];
    d.bnd[k] = (IDX)g.bnd[k];
    d.fdm[k] = g.fdm[k];
    d.fds[k] = g.fds[k];
    d.lg[k] = g.lg[k];
  }
  d.pow2 = g.pow2 ? 1u : 0u;
  d.lin0 = (IDX)g.lin0;
  d.nvec = (IDX)g.nvec;
  d.nelem = (IDX)g.N;
  d.wmul = (IDX)g.wmul;
  d.wspan = (IDX)g.wspan;
  d.dv = (IDX)g.dv;
  d.khi = g.khi;
  d.klo = g.klo;
  d.lgL = (uint32_t)g.lgL;
  d.R = (uint32_t)g.R;
  d.rowmul = (IDX)g.rowmul;
  d.colmul = (IDX)g.colmul;
  d.vfull = (IDX)g.vfull;
  d.vany = (IDX)g.vany;
  d.srows = (IDX)g.srows;
  d.scols = (IDX)g.scols;
  d.collapsed = g.collapsed ? 1 : 0;
  d.d_out = g.nout >= 0 ? g.nout : g.d + (g.with_mass ? 1 : 0);
  d.op = g.binop;
  d.split = g.split ? 1 : 0;
  d.cluster = g.cluster;
  d.nax = g.nax;
  for (int k = 0; k < TRIOT_MAXD; ++k) d.offd[k] = g.offd[k];
  d.zmask = g.zmask;
  d.rowlen = (uint32_t)g.rowlen;
  d.rmag = (uint32_t)g.rmag;
  d.rwin = (uint32_t)g.rwin;
  d.dshift = g.dshift;
  d.evpad = g.evpad ? 1u : 0u;
  d.seglen = (IDX)g.seglen;
  d.segm = (IDX)g.segm;
  for (int k = 0; k < TRIOT_MAXD; ++k) {
    d.zn[k] = (IDX)g.zn[k];
    d.zdm[k] = g.zdm[k];
    d.zds[k] = g.zds[k];
  }
  for (int x = 0; x < TRIOT_MAXT; ++x) {
    for (int k = 0; k < TRIOT_MAXD; ++k) {
      d.t[x].sig[k] = (IDX)g.t[x].sig[k];
      d.t[x].kap[k] = (IDX)g.t[x].kap[k];
    }
    d.t[x].step = (IDX)g.t[x].step;
    d.t[x].rho = (IDX)g.t[x].rho;
    d.t[x].tau = (IDX)g.t[x].tau;
    d.t[x].vec = g.t[x].vec ? 1u : 0u;
    d.t[x].numel_pad = 0;
    d.t[x].ptr = g.t[x].ptr;
  }
  d.out = nullptr;
  d.ws = nullptr;
}

}  // namespace triot
