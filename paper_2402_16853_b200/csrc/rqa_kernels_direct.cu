// Direct-evaluation kernels (runtime m, tau; no term reuse) and the m = 1
// kernel (|d| <= radius for every metric, embedding.py:88-89,144-147).
#include "rqa_variants.cuh"

namespace rqa {

bool find_variant_m1(int m, int tau, bool small, Variant* out) {
  (void)tau;
  if (m != 1) return false;
  *out = small ? make_variant<kL1, 1, 1, 4, 2>(0) : make_variant<kL1, 1, 1, 8, 4>(0);
  return true;
}

bool find_variant_direct(int metric, int m, int tau, bool small, Variant* out) {
  const long long w = (long long)(m - 1) * tau;
  if (w > 4096) return false;  // shared-memory windows would not fit
  const int wi = (int)w;
  if (small) {
    switch (metric) {
      case kL1: *out = make_variant<kL1, 0, 1, 4, 2>(wi); return true;
      case kL2: *out = make_variant<kL2, 0, 1, 4, 2>(wi); return true;
      case kLinf: *out = make_variant<kLinf, 0, 1, 4, 2>(wi); return true;
    }
  }
  switch (metric) {
    case kL1: *out = make_variant<kL1, 0, 1, 8, 4>(wi); return true;
    case kL2: *out = make_variant<kL2, 0, 1, 8, 4>(wi); return true;
    case kLinf: *out = make_variant<kLinf, 0, 1, 8, 4>(wi); return true;
  }
  return false;
}

}  // namespace rqa
