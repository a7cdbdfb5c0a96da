// Sparse-prefilter instantiations (PREC = 2, exact float64): L2 / L1 term
// reuse replaced by the AND of per-component predicates |d| <= D* plus exact
// sums for the candidate cells (rqa_unit.cuh, kPre).
#include "rqa_variants.cuh"

namespace rqa {

bool find_variant_pre(int metric, int m, int tau, Variant* out) {
#define RQA_CASE(MET, MM, TT)                                              \
  if (metric == MET && m == MM && tau == TT) {                             \
    *out = make_variant<MET, MM, TT, 8, 4, 2>(0);                          \
    return true;                                                           \
  }
  RQA_CASE(kL2, 2, 1) RQA_CASE(kL2, 2, 2) RQA_CASE(kL2, 2, 3) RQA_CASE(kL2, 3, 1)
  RQA_CASE(kL2, 3, 2) RQA_CASE(kL2, 3, 3) RQA_CASE(kL2, 4, 1) RQA_CASE(kL2, 4, 2)
  RQA_CASE(kL2, 5, 1) RQA_CASE(kL1, 2, 1) RQA_CASE(kL1, 2, 2) RQA_CASE(kL1, 3, 1)
  // large windows: the float64 term window would need one slot per lane
  // (R = 1, 8 warps per SM); the prefilter keeps only predicate bits
  RQA_CASE(kL1, 10, 5) RQA_CASE(kL2, 10, 5) RQA_CASE(kL1, 5, 5) RQA_CASE(kL2, 5, 5)
#undef RQA_CASE
  return false;
}

}  // namespace rqa
