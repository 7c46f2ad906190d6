// inst.cu -- explicit instantiation of one kernel family and its dispatch table.
//
// Compiled several times with different macros (build.py), one object per (op, element size,
// binary op), so the D = 1..16 x V x IDX matrix compiles in parallel -- the GPU analogue of the
// paper's compile-time note (max dimension 16 compiles in 16 s).  The table replaces
// LinearTemplateSearch (Alg 7): runtime (D, V, index width) -> kernel in O(1).
//
//   TRIOT_INST_OP   0 = embed, 1 = binary, 2 = expected value, 3 = inner product,
//                   4 = fused update, 5 = naive convolution
//   TRIOT_INST_ESZ  4 or 8
//   TRIOT_INST_BOP  binary op 0..3 (binary); 1 = bulk-copy variant, 2 = views (expected value)
#include "kernels.cuh"

#ifndef TRIOT_INST_OP
#error "define TRIOT_INST_OP"
#endif
#ifndef TRIOT_INST_ESZ
#error "define TRIOT_INST_ESZ"
#endif
#ifndef TRIOT_INST_BOP
#define TRIOT_INST_BOP 0
#endif

#define TRIOT_CAT2(a, b) a##b
#define TRIOT_CAT(a, b) TRIOT_CAT2(a, b)
#define TRIOT_NAME \
  TRIOT_CAT(TRIOT_CAT(TRIOT_CAT(triot_table_, TRIOT_INST_OP), TRIOT_CAT(_, TRIOT_INST_ESZ)), \
            TRIOT_CAT(_, TRIOT_INST_BOP))

namespace triot {
namespace {

constexpr int ESZ = TRIOT_INST_ESZ;

// loads in flight per lane per batch (bytes in flight, SURVEY §8(d) Little's law)
constexpr int KEMBED = 4;
constexpr int KBIN = 2;
constexpr int KEV = 2;

template <int D, int V, typename IDX>
const void* kptr() {
  // One-element vectors are never planned for embed, binary or the dense expected value: an
  // innermost extent no vector width divides takes flat vectors (plan.cpp: flat_ok) or row
  // windows instead -- so those instances are not compiled (tests/test_boundary_cpu.py
  // test_planner_never_selects_uncompiled_instances).  Dot, update, convolution and the EV of
  // a view keep them.
#if TRIOT_INST_OP == 0 || TRIOT_INST_OP == 1 || (TRIOT_INST_OP == 2 && TRIOT_INST_BOP == 0)
  constexpr bool kSkip = V == 1;
#else
  constexpr bool kSkip = false;
#endif
  if constexpr (kSkip) {
    return nullptr;
  } else {
#if TRIOT_INST_OP == 0
  return (const void*)&embed_kernel<D, ESZ, V, IDX, KEMBED, false>;
#elif TRIOT_INST_OP == 1
  return (const void*)&binary_kernel<D, ESZ, V, IDX, KBIN, TRIOT_INST_BOP>;
#elif TRIOT_INST_OP == 3
  return (const void*)&dot_kernel<D, ESZ, V, IDX, KBIN>;
#elif TRIOT_INST_OP == 4
  return (const void*)&update_kernel<D, ESZ, V, IDX, KBIN>;
#elif TRIOT_INST_OP == 5
  // naive convolution, idx64 slot = the shared-memory staged variant: vi 2 (V = 1) = the group
  // kernel, vi 0 / 1 (the V = 32 / 16 byte slots) = the lane-per-output kernel forward / reversed
  constexpr bool S = sizeof(IDX) == 8;
  if (V == 1) return (const void*)&conv_kernel<D, ESZ, S>;
  if (V == 32 / ESZ) return (const void*)&conv_lane_kernel<D, ESZ, S, false>;
  return (const void*)&conv_lane_kernel<D, ESZ, S, true>;
#elif TRIOT_INST_BOP == 2
  // expected value of a view (strided p)
  return (const void*)&ev_view_kernel<D, ESZ, V, IDX, KEV>;
#elif TRIOT_INST_BOP == 1
  // EV bulk-copy fast path: only the 32-byte vector width exists; vi slot 1 (16 B) carries the
  // small-stage variant
  if (V == 32 / ESZ) return (const void*)&ev_tma_kernel<D, ESZ, IDX>;
  if (V == 16 / ESZ)
    return (const void*)&ev_tma_kernel<D, ESZ, IDX, TRIOT_EVS_NSTAGE, TRIOT_EVS_SVEC,
                                       TRIOT_EVS_BLOCK>;
  return nullptr;
#else
  return (const void*)&ev_kernel<D, ESZ, V, IDX, KEV>;
#endif
  }
}

// flat-vector instances (odd innermost extents): embed, binary, expected value
template <int D, typename IDX>
const void* kptr_flat() {
#if TRIOT_INST_OP == 0
  return (const void*)&embed_flat_kernel<D, ESZ, IDX, 2>;
#elif TRIOT_INST_OP == 1
  return (const void*)&binary_flat_kernel<D, ESZ, IDX, 2, TRIOT_INST_BOP>;
#elif TRIOT_INST_OP == 2 && TRIOT_INST_BOP == 0
  return (const void*)&ev_flat_kernel<D, ESZ, IDX, 2>;
#else
  return nullptr;
#endif
}

// row-window instances (short odd innermost extents): embed, binary; K = 32 bytes of loads per
// lane per batch (measured on B200: f32 K 8 > 4, f64 K 4 > 8); the dense expected value's
// shared-memory row tiles (D = the outer axes, at most 15)
template <int D, typename IDX>
const void* kptr_rows() {
#if TRIOT_INST_OP == 0
  return (const void*)&embed_rows_kernel<D, ESZ, IDX, 32 / ESZ>;
#elif TRIOT_INST_OP == 1
  return (const void*)&binary_rows_kernel<D, ESZ, IDX, 32 / ESZ, TRIOT_INST_BOP>;
#elif TRIOT_INST_OP == 2 && TRIOT_INST_BOP == 0
  if constexpr (D >= TRIOT_MAXD) {
    return nullptr;
  } else {
    return (const void*)&ev_rows_kernel<D, ESZ, IDX>;
  }
#else
  return nullptr;
#endif
}

// row windows, warp per row (long rows): embed, binary
template <int D, typename IDX>
const void* kptr_rowsw() {
#if TRIOT_INST_OP == 0
  return (const void*)&embed_rowsw_kernel<D, ESZ, IDX>;
#elif TRIOT_INST_OP == 1
  return (const void*)&binary_rowsw_kernel<D, ESZ, IDX, TRIOT_INST_BOP>;
#elif TRIOT_INST_OP == 2 && TRIOT_INST_BOP == 0
  // the expected value has no warp-per-row kernel: the slot carries its flat 64-byte units
  return (const void*)&ev_flat_kernel<D, ESZ, IDX, 1, 64>;
#else
  return nullptr;
#endif
}

// embed / binary into a misaligned output dense in the counter (shifted 32-B stores)
template <int D, typename IDX>
const void* kptr_shift() {
#if TRIOT_INST_OP == 0
  return (const void*)&embed_shift_kernel<D, ESZ, IDX, KEMBED>;
#elif TRIOT_INST_OP == 1
  return (const void*)&binary_shift_kernel<D, ESZ, IDX, KBIN, TRIOT_INST_BOP>;
#else
  return nullptr;
#endif
}

// embed with zero runs (32-B vectors, dst dense in the counter; Desc::zmask)
template <int D, typename IDX>
const void* kptr_zero_runs() {
#if TRIOT_INST_OP == 0
  if constexpr (D < 2) {  // zero runs need an outer digit khi < D - 1 (plan.cpp set_step)
    return nullptr;
  } else {
    return (const void*)&embed_kernel<D, ESZ, 32 / ESZ, IDX, KEMBED, true>;
  }
#else
  return nullptr;
#endif
}

// table index: ((D-1) * NVI + vi) * 2 + idx64, vi: 0 = 32 B, 1 = 16 B, 2 = one element,
// 3 = flat 32-B vectors, 4 = 32 B with embed zero runs, 5 = row windows, 6 = row windows with
// a warp per row (expected value: flat 64-byte units), 7 = 32 B with shifted stores (embed into a misaligned dense dst)
constexpr int NVI = 8;
template <int D>
struct Fill {
  static void run(const void** t) {
    t[((D - 1) * NVI + 7) * 2 + 0] = kptr_shift<D, uint32_t>();
    t[((D - 1) * NVI + 7) * 2 + 1] = kptr_shift<D, uint64_t>();
    t[((D - 1) * NVI + 6) * 2 + 0] = kptr_rowsw<D, uint32_t>();
    t[((D - 1) * NVI + 6) * 2 + 1] = kptr_rowsw<D, uint64_t>();
    t[((D - 1) * NVI + 5) * 2 + 0] = kptr_rows<D, uint32_t>();
    t[((D - 1) * NVI + 5) * 2 + 1] = kptr_rows<D, uint64_t>();
    t[((D - 1) * NVI + 4) * 2 + 0] = kptr_zero_runs<D, uint32_t>();
    t[((D - 1) * NVI + 4) * 2 + 1] = kptr_zero_runs<D, uint64_t>();
    t[((D - 1) * NVI + 0) * 2 + 0] = kptr<D, 32 / ESZ, uint32_t>();
    t[((D - 1) * NVI + 0) * 2 + 1] = kptr<D, 32 / ESZ, uint64_t>();
    t[((D - 1) * NVI + 1) * 2 + 0] = kptr<D, 16 / ESZ, uint32_t>();
    t[((D - 1) * NVI + 1) * 2 + 1] = kptr<D, 16 / ESZ, uint64_t>();
    t[((D - 1) * NVI + 2) * 2 + 0] = kptr<D, 1, uint32_t>();
    t[((D - 1) * NVI + 2) * 2 + 1] = kptr<D, 1, uint64_t>();
    t[((D - 1) * NVI + 3) * 2 + 0] = kptr_flat<D, uint32_t>();
    t[((D - 1) * NVI + 3) * 2 + 1] = kptr_flat<D, uint64_t>();
    Fill<D - 1>::run(t);
  }
};
template <>
struct Fill<0> {
  static void run(const void**) {}
};

struct Table {
  const void* t[TRIOT_MAXD * NVI * 2];
  Table() { Fill<TRIOT_MAXD>::run(t); }
};

}  // namespace
}  // namespace triot

extern "C" const void* TRIOT_NAME(int D, int vi, int idx64) {
  static const triot::Table tab;  // thread-safe one-time init
  if (D < 1 || D > TRIOT_MAXD || vi < 0 || vi >= triot::NVI) return nullptr;
  return tab.t[((D - 1) * triot::NVI + vi) * 2 + (idx64 ? 1 : 0)];
}
