// f32 filter instantiations (PREC = 1): packed f32x2 L1 term reuse, and the
// direct f32 kernels for every other metric / embedding (rqa_unit.cuh).
#include "rqa_variants.cuh"

namespace rqa {

bool find_variant_f32_l1(int m, int tau, Variant* out) {
#define RQA_CASE(MM, TT)                                                   \
  if (m == MM && tau == TT) {                                              \
    *out = make_variant<kL1, MM, TT, 8, 4, 1>(0);                         \
    return true;                                                           \
  }
  RQA_CASE(2, 1) RQA_CASE(2, 2) RQA_CASE(2, 3) RQA_CASE(3, 1) RQA_CASE(3, 2)
  RQA_CASE(3, 3) RQA_CASE(4, 1) RQA_CASE(4, 2) RQA_CASE(5, 1)
#undef RQA_CASE
  // large windows: one slot pair per lane
  if (m == 10 && tau == 5) { *out = make_variant<kL1, 10, 5, 8, 2, 1>(0); return true; }
  if (m == 5 && tau == 5) { *out = make_variant<kL1, 5, 5, 8, 2, 1>(0); return true; }
  return false;
}

bool find_variant_f32_direct(int metric, int m, int tau, Variant* out) {
  const long long w = (long long)(m - 1) * tau;
  if (w > 4096) return false;
  switch (metric) {
    case kL1: *out = make_variant<kL1, 0, 1, 8, 4, 1>((int)w); return true;
    case kL2: *out = make_variant<kL2, 0, 1, 8, 4, 1>((int)w); return true;
    case kLinf: *out = make_variant<kLinf, 0, 1, 8, 4, 1>((int)w); return true;
  }
  return false;
}

}  // namespace rqa
