// Reuse-kernel instantiations for metric linf, 256-row bands (NW = 4, R = 2).
#include "rqa_variants.cuh"

namespace rqa {

bool find_variant_linf_small(int m, int tau, Variant* out) {
#define RQA_CASE(MM, TT)                                                   \
  if (m == MM && tau == TT) {                                              \
    *out = make_variant<kLinf, MM, TT, 4, 2>(0);                            \
    return true;                                                           \
  }
  RQA_CASE(2, 1) RQA_CASE(2, 2) RQA_CASE(3, 1) RQA_CASE(3, 2) RQA_CASE(4, 1)
#undef RQA_CASE
  return false;
}

}  // namespace rqa
