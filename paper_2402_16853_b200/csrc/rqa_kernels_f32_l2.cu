// f32 filter instantiations (PREC = 1): packed f32x2 L2 term reuse.
#include "rqa_variants.cuh"

namespace rqa {

bool find_variant_f32_l2(int m, int tau, Variant* out) {
#define RQA_CASE(MM, TT)                                                   \
  if (m == MM && tau == TT) {                                              \
    *out = make_variant<kL2, MM, TT, 8, 4, 1>(0);                         \
    return true;                                                           \
  }
  RQA_CASE(2, 1) RQA_CASE(2, 2) RQA_CASE(2, 3) RQA_CASE(3, 1) RQA_CASE(3, 2)
  RQA_CASE(3, 3) RQA_CASE(4, 1) RQA_CASE(4, 2) RQA_CASE(5, 1)
#undef RQA_CASE
  if (m == 10 && tau == 5) { *out = make_variant<kL2, 10, 5, 8, 2, 1>(0); return true; }
  if (m == 5 && tau == 5) { *out = make_variant<kL2, 5, 5, 8, 2, 1>(0); return true; }
  return false;
}

}  // namespace rqa
