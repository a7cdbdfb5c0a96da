// Reuse-kernel instantiations for metric linf, 1024-row bands (see rqa_sym.cuh).
#include "rqa_variants.cuh"

namespace rqa {

// 256-row geometry: only through RQA_GEOMETRY=small (work units balance any n)
static bool find_variant_linf_small(int, int, Variant*) { return false; }

bool find_variant_linf(int m, int tau, bool small, Variant* out) {
  if (small && find_variant_linf_small(m, tau, out)) return true;
#define RQA_CASE(MM, TT)                                                   \
  if (m == MM && tau == TT) {                                              \
    *out = make_variant<kLinf, MM, TT, 8, 4>(0);                            \
    return true;                                                           \
  }
  RQA_CASE(2, 1) RQA_CASE(2, 2) RQA_CASE(2, 3) RQA_CASE(3, 1) RQA_CASE(3, 2)
  RQA_CASE(3, 3) RQA_CASE(4, 1) RQA_CASE(4, 2) RQA_CASE(5, 1)
#undef RQA_CASE

  return false;
}

}  // namespace rqa
