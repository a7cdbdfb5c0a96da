// Reuse-kernel instantiations for metric l2, 1024-row bands (see rqa_sym.cuh).
#include "rqa_variants.cuh"

namespace rqa {

// 256-row geometry: only through RQA_GEOMETRY=small (work units balance any n)
static bool find_variant_l2_small(int, int, Variant*) { return false; }

bool find_variant_l2(int m, int tau, bool small, Variant* out) {
  if (small && find_variant_l2_small(m, tau, out)) return true;
#define RQA_CASE(MM, TT)                                                   \
  if (m == MM && tau == TT) {                                              \
    *out = make_variant<kL2, MM, TT, 8, 4>(0);                            \
    return true;                                                           \
  }
  RQA_CASE(2, 1) RQA_CASE(2, 2) RQA_CASE(2, 3) RQA_CASE(3, 1) RQA_CASE(3, 2)
  RQA_CASE(3, 3) RQA_CASE(4, 1) RQA_CASE(4, 2) RQA_CASE(5, 1)
#undef RQA_CASE
  // large windows: one slot per lane, the term window lives in registers
  if (m == 10 && tau == 5) { *out = make_variant<kL2, 10, 5, 8, 1>(0); return true; }
  if (m == 5 && tau == 5) { *out = make_variant<kL2, 5, 5, 8, 1>(0); return true; }
  return false;
}


}  // namespace rqa
