// rqa_variants.cuh -- compile-time kernel variants and their launchers.
#pragma once
#include <cstdlib>

#include "rqa_sym.cuh"
#include "rqa_unit.cuh"

namespace rqa {

struct Variant {
  int nw, r;              // warps per CTA, stacked slots (band = r * 32 * nw rows)
  int w;                  // term window (m-1)*tau
  int reuse;              // 1: compile-time (m, tau) with term reuse; 0: direct
  int prec;               // 0: float64 evaluation; 1: f32 filter; 2: prefilter (rqa_unit.cuh)
  size_t smem;            // dynamic shared memory bytes
  int f32pred;            // prefilter with the packed float32 component predicate
  cudaError_t (*launch)(const UnitArgs&, int nunits, int w, cudaStream_t);
  const void* kernel;     // for occupancy queries
  int64_t band_rows() const { return (int64_t)r * 32 * nw; }
  int64_t slot_rows() const { return (int64_t)32 * nw; }
};

// 2 CTAs per SM, except the one-slot (pair) large-window variants (registers).
template <int M, int TAU, int NW, int R>
constexpr int min_blocks() {
  return (R <= 2 && M > 0 && (M - 1) * TAU > 16) ? 1 : (NW == 4 ? 4 : (R == 2 ? 3 : 2));
}

template <int METRIC, int M, int TAU, int NW, int R, int PREC = 0>
cudaError_t launch_unit(const UnitArgs& a, int nunits, int w, cudaStream_t st) {
  const SymSmem L(NW, R, M == 0 ? w : (M - 1) * TAU, PREC == 1 ? 4 : 8, kCandCapOf<PREC, M>,
                  kF32Pred<PREC, M, R>);
  auto k = unit_kernel<METRIC, M, TAU, NW, R, min_blocks<M, TAU, NW, R>(), PREC>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
  if (e != cudaSuccess) return e;
  k<<<nunits, NW * 32, L.total, st>>>(a, w);
  return cudaGetLastError();
}

template <int METRIC, int M, int TAU, int NW, int R, int PREC = 0>
Variant make_variant(int w_rt) {
  const int w = (M == 0) ? w_rt : (M - 1) * TAU;
  const SymSmem L(NW, R, w, PREC == 1 ? 4 : 8, kCandCapOf<PREC, M>, kF32Pred<PREC, M, R>);
  return Variant{NW, R, w, M == 0 ? 0 : 1, PREC, L.total, kF32Pred<PREC, M, R> ? 1 : 0,
                 &launch_unit<METRIC, M, TAU, NW, R, PREC>,
                 (const void*)&unit_kernel<METRIC, M, TAU, NW, R, min_blocks<M, TAU, NW, R>(),
                                           PREC>};
}

// Implemented in rqa_kernels_<metric>[_small].cu (one translation unit each so
// the instantiations compile in parallel).  `small` selects the 256-row band
// geometry (NW = 4, R = 2) used when the 1024-row bands would be too few to
// balance the SMs (the upper triangle makes early bands the largest).
bool find_variant_l1(int m, int tau, bool small, Variant* out);
bool find_variant_l2(int m, int tau, bool small, Variant* out);
bool find_variant_linf(int m, int tau, bool small, Variant* out);
bool find_variant_m1(int m, int tau, bool small, Variant* out);
bool find_variant_direct(int metric, int m, int tau, bool small, Variant* out);
// f32 filter kernels (PREC = 1): packed L1/L2 term reuse, else direct.
bool find_variant_f32_l1(int m, int tau, Variant* out);
bool find_variant_f32_l2(int m, int tau, Variant* out);
bool find_variant_f32_direct(int metric, int m, int tau, Variant* out);

// Sparse prefilter kernels (PREC = 2, exact; rqa_unit.cuh kPre).
bool find_variant_pre(int metric, int m, int tau, Variant* out);

inline bool find_variant_f32(int metric, int m, int tau, bool packed_only, Variant* out) {
  if (m >= 2 && metric == kL1 && find_variant_f32_l1(m, tau, out)) return true;
  if (m >= 2 && metric == kL2 && find_variant_f32_l2(m, tau, out)) return true;
  return !packed_only && find_variant_f32_direct(metric, m, tau, out);
}

// Rows below which the 256-row geometry is chosen.  Work units balance the
// SMs for any n, so the 1024-row geometry is used everywhere by default.
constexpr int64_t kSmallGeometryBelow = 0;

inline bool find_variant(int metric, int m, int tau, int64_t n, Variant* out) {
  // RQA_GEOMETRY=small|big overrides the choice (benchmarking / tests)
  static const char* force = getenv("RQA_GEOMETRY");
  const bool small = force && force[0] == 's' ? true
                   : force && force[0] == 'b' ? false
                                              : n < kSmallGeometryBelow;

  if (m == 1) return find_variant_m1(m, tau, small, out);
  bool ok = false;
  if (metric == kL1) ok = find_variant_l1(m, tau, small, out);
  else if (metric == kL2) ok = find_variant_l2(m, tau, small, out);
  else if (metric == kLinf) ok = find_variant_linf(m, tau, small, out);
  return ok || find_variant_direct(metric, m, tau, small, out);
}

}  // namespace rqa
