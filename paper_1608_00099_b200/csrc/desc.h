// desc.h -- the launch descriptor: a POD built on the host (plan.cpp) and passed by value as a
// kernel parameter (< 2 KB, lives in the constant parameter bank, so every field read in the
// kernels is a constant-bank operand, not a load).
//
// Vocabulary:
//   counter    the iteration shape (dst for embed, iter for binary, p for EV), after
//              canonicalisation (unit axes dropped, contiguous axes merged).
//   vector     V consecutive counter elements (32 bytes when geometry and alignment allow).
//   flat       (odd innermost extents) vectors of V consecutive elements of the flattened
//              counter that may cross rows: digits are then element digits (D = all axes) and
//              the kernel walks the V elements with the +1 odometer.
//   rows       (short odd innermost extents, embed / binary) a vector is one counter row; the
//              digits are the outer axes and a warp sweeps its 32 rows' elements lane by lane.
//   digits     u[0..D-1]: the mixed-radix coordinates of a vector.  Digits 0..D-2 are counter
//              axes; digit D-1 (the "vector digit") is either the vector index inside a counter
//              row (R == 1) or a group of R whole rows when rows are shorter than a vector
//              (R > 1: the inner-axis collapse for tiny innermost extents).
//   step       +32 vectors (one warp-wide stride), pre-decoded into mixed-radix digits dlt[].
//   sig[k]     a tensor's Horner stride of digit k (Alg 2 / P:50 applied to its own shape).
//   kap[k]     the offset change when digit k carries out: sig[k-1] - ext[k] * sig[k].
#pragma once
#include <stdint.h>

#define TRIOT_MAXD 16
#define TRIOT_MAXT 3
#define TRIOT_BLOCK 256   // threads per block of the streaming kernels
#define TRIOT_CONV_BLOCK 128  // convolution: threads per block
#define TRIOT_CONV_GROUP 8    // convolution, group kernel: lanes per output

namespace triot {

enum Op { OP_EMBED = 0, OP_BINARY = 1, OP_EV = 2, OP_DOT = 3, OP_UPDATE = 4, OP_CONV = 5 };

template <typename IDX>
struct TensorAcc {
  IDX sig[TRIOT_MAXD];   // stride (elements) of each vector digit
  IDX kap[TRIOT_MAXD];   // carry delta of each digit (kap[0] unused)
  IDX step;              // offset change of a +32-vector step, before carries
  IDX rho;               // stride of the row inside a collapsed vector (R > 1)
  IDX tau;               // stride of the innermost counter axis (1 for contiguous rows)
  uint32_t vec;          // 1: V elements are contiguous and V*esz-aligned -> one wide access
  uint32_t numel_pad;    // convolution: operand elements rounded up (shared-memory layout)
  const void* ptr;       // device base pointer
};

template <typename IDX>
struct Desc {
  IDX ext[TRIOT_MAXD];   // digit extents
  IDX dlt[TRIOT_MAXD];   // digits of the +32-vector step
  IDX bnd[TRIOT_MAXD];   // embed: digit k (k < D-1) is in bounds iff u[k] < bnd[k]
  uint32_t fdm[TRIOT_MAXD];  // fast-division magic multiplier per digit extent (IDX = u32)
  uint32_t fds[TRIOT_MAXD];  // fast-division shifts: s1 | s2 << 8
  uint32_t pow2;             // 1: every digit extent 1..D-1 is a power of two (decode by shifts)
  uint8_t lg[TRIOT_MAXD];    // log2 of each digit extent when pow2
  IDX lin0;                  // tensor 0 offset of digit vector index v is v * lin0 (0: use Horner)
  IDX nvec;              // number of vectors W
  IDX nelem;             // counter elements N (flat vectors: the last vector may be partial)
  // work decomposition: warp w starts at vector w*wmul + lane, owns
  // the window [w*wmul, min(w*wmul + wspan, W)) and advances by dv vectors per step.
  //   chunk mode:  wmul = wspan = Q*32, dv = 32      (each warp streams a contiguous run)
  //   stride mode: wmul = 32, wspan = W, dv = 32*warps (all warps sweep one window together)
  IDX wmul, wspan, dv;
  int32_t khi, klo;      // innermost / outermost digit with a nonzero step digit
  // in-vector geometry
  uint32_t lgL;          // log2(elements per row inside a vector): log2(V) if R == 1
  uint32_t R;            // rows per vector
  IDX rowmul, colmul;    // first row / col of a vector = u[D-1] * rowmul / colmul
  IDX vfull, vany;       // embed: vector digit u fully in bounds iff u < vfull, any iff u < vany
  IDX srows, scols;      // embed: per-element bounds of a partial vector
  // expected value: weight slots -> output
  int32_t collapsed;     // 1 iff R > 1
  int32_t d_out;         // values written: the caller's d (+1 when the mass is requested)
  int32_t slot_of_axis[TRIOT_MAXD + 1];  // out[j] = slot >= 0 ? total[slot] : 0 (slot D+1 = mass)
  int32_t op;            // binary op
  int32_t split;         // reductions: 1 = write the block partial only; ev_final_kernel sums
  uint32_t cluster;      // reductions: > 1 = the grid is ONE thread-block cluster of this many
                         // blocks; the partials meet in block 0's shared memory (DSMEM)
  // expected value of a block of a larger PMF (slab / chunk / shard): output axis j < nax
  // gets offd[j] * mass added (global coordinate = offset + local), mass = slot_of_axis[nax]
  int32_t nax;
  double offd[TRIOT_MAXD];
  // embed zero runs: 32 vectors == one unit of digit khi (lanes share digits 0..khi) and dst is
  // dense in the counter, so while a digit <= khi is out of bounds the warp stores zeros at
  // dst + r * step without touching the odometer (zmask = oob bits of digits 0..khi, 0 = off)
  uint32_t zmask;
  // zero-run lengths: zn[m] = size of the sub-counter of digits m..khi (its value is the warp's
  // step index mod zn[m]), with fast-division magics
  uint32_t zdm[TRIOT_MAXD], zds[TRIOT_MAXD];
  IDX zn[TRIOT_MAXD];
  // row windows (short odd innermost extents, embed / binary): a vector is one counter row of
  // rowlen elements; a warp sweeps groups of rwin windows of 32 rows, element e of a group in
  // lane e % 32, row umulhi(e, rmag) = e / rowlen (rmag = 2^32 / rowlen + 1, exact for
  // e < 2^13); scols = the embed bound of the column.
  uint32_t rowlen, rmag, rwin;
  // expected value row tiles: 1 = a thread takes rwin consecutive rows of a tile (+1 digit steps
  // between them, the step dlt to its group in the next tile); 0 = rows t, t + block, ...
  uint32_t rgroup;
  // rows that are segments of a longer split axis (seglen = rowlen): the embed bound of the
  // unsplit axis is segm, so segment s reads columns [0, clamp(segm - s rowlen, 0, rowlen))
  IDX seglen, segm;
  // embed into a dst dense in the counter whose base is misaligned by dshift elements (> 0):
  // aligned 32-byte stores of lane-shifted vectors (embed_shift_kernel)
  uint32_t dshift;
  // EV of a view with odd rows: vectors padded past the row end; elements at column >= scols
  // (row length) read as +0
  uint32_t evpad;
  TensorAcc<IDX> t[TRIOT_MAXT];   // embed: dst, src; binary: c, a, b; EV: p; dot: a, b;
                                  // update: x, y, z
  void* out;             // EV: means (device)
  void* ws;              // EV: workspace (device)
};

// Workspace layout of the reductions (expected value, inner product):
//   [arrival counter u32 | pad to 256 B] [grid x P block partials]   (P = slots per block)
// Zero-filled once by the caller; every call leaves the counter at 0.
#define TRIOT_EV_MAX_GRID 8192
#define TRIOT_CLUSTER_MAX 8   // blocks of a one-cluster reduction (the portable cluster size)
#define TRIOT_EV_WS_HEADER 256
// EV bulk-copy pipeline: NSTAGE shared-memory stages of SVEC 32-byte vectors per block
#define TRIOT_EV_NSTAGE 6
#define TRIOT_EV_SVEC 1024
#define TRIOT_EV_TMA_BLOCK 512
#define TRIOT_EV_SMEM (TRIOT_EV_NSTAGE * TRIOT_EV_SVEC * 32 + 2 * TRIOT_EV_NSTAGE * 8)
// the small-stage variant: several resident blocks per SM, many blocks per launch (the hardware
// block scheduler balances the SMs; each block's partial keeps the sum deterministic)
#define TRIOT_EVS_NSTAGE 4
#define TRIOT_EVS_SVEC 512
#define TRIOT_EVS_BLOCK 256
#define TRIOT_EVS_SMEM (TRIOT_EVS_NSTAGE * TRIOT_EVS_SVEC * 32 + 2 * TRIOT_EVS_NSTAGE * 8)

}  // namespace triot
