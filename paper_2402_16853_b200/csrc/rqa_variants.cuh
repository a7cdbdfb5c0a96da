// rqa_variants.cuh -- compile-time kernel variants and their launchers.
#pragma once
#include "rqa_band.cuh"

namespace rqa {

struct Variant {
  int nw, r, hs;          // warps per CTA, stacked slots, slot height
  int w;                  // term window (m-1)*tau
  int reuse;              // 1: compile-time (m, tau) with term reuse; 0: direct
  size_t smem;            // dynamic shared memory bytes
  cudaError_t (*launch)(const BandArgs&, int nbands, int w, cudaStream_t);
  int64_t band_rows() const { return (int64_t)r * hs; }
};

template <int METRIC, int M, int TAU, int NW, int R, int HS>
cudaError_t launch_band(const BandArgs& a, int nbands, int w, cudaStream_t st) {
  using C = BandCfg<METRIC, M, TAU, NW, R, HS>;
  const BandSmem L(NW, R, HS, C::kDirect ? w : C::kW);
  auto k = band_kernel<METRIC, M, TAU, NW, R, HS>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
  if (e != cudaSuccess) return e;
  k<<<nbands, NW * 32, L.total, st>>>(a, w);
  return cudaGetLastError();
}

template <int METRIC, int M, int TAU, int NW, int R, int HS>
Variant make_variant(int w_rt) {
  using C = BandCfg<METRIC, M, TAU, NW, R, HS>;
  const int w = C::kDirect ? w_rt : C::kW;
  const BandSmem L(NW, R, HS, w);
  return Variant{NW, R, HS, w, C::kDirect ? 0 : 1, L.total, &launch_band<METRIC, M, TAU, NW, R, HS>};
}

// Implemented in rqa_kernels_<metric>.cu (one translation unit per metric so
// the instantiations compile in parallel).
bool find_variant_l1(int m, int tau, Variant* out);
bool find_variant_l2(int m, int tau, Variant* out);
bool find_variant_linf(int m, int tau, Variant* out);
bool find_variant_m1(int m, int tau, Variant* out);
bool find_variant_direct(int metric, int m, int tau, Variant* out);

inline bool find_variant(int metric, int m, int tau, Variant* out) {
  if (m == 1) return find_variant_m1(m, tau, out);
  bool ok = false;
  if (metric == kL1) ok = find_variant_l1(m, tau, out);
  else if (metric == kL2) ok = find_variant_l2(m, tau, out);
  else if (metric == kLinf) ok = find_variant_linf(m, tau, out);
  return ok || find_variant_direct(metric, m, tau, out);
}

}  // namespace rqa
