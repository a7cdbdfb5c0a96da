// rqa_fold.cuh -- stitches diagonal runs across band / stripe boundaries.
//
// Every segment g of rows [lo_g, hi_g) reports, per diagonal k >= 0, the
// length of the 1-run starting at its top edge (P) and ending at its bottom
// edge (S); runs touching neither edge were already counted by the band
// kernel.  Folding the segments of one diagonal in row order is the
// reference's carry-over contract (engine.py:287-319: absorb the incoming
// carry, count finished runs, count a "stale" carry, write back an open run)
// and flush (engine.py:195-212), applied to whole segments instead of tiles.
// Diagonal k > 0 counts twice: R = R^T makes diagonal -k identical.
#pragma once
#include "rqa_device.cuh"

namespace rqa {

enum FoldMode : int { kFoldFinal = 0, kFoldStripe = 1 };

template <typename TS>
struct FoldArgs {
  const TS* P;              // [nseg][pitch]
  const TS* S;              // [nseg][pitch]
  int64_t pitch;
  const int64_t* bounds;    // nseg+1 row boundaries (device)
  int nseg;
  int64_t n;
  unsigned long long* hist; // [3][n+1] (only the diagonal part is touched)
  int32_t* out_p;           // stripe mode: prefix of the whole stripe per k
  int32_t* out_s;           // stripe mode: suffix of the whole stripe per k
};

template <typename TS>
__global__ void fold_kernel(const FoldArgs<TS> a, const int mode) {
  const int64_t n = a.n;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long wgt = (k == 0) ? 1ull : 2ull;
    const int64_t rows = n - k;  // diagonal k has rows [0, n-k)
    int64_t open = 0;
    int64_t pstr = -1;
    for (int g = 0; g < a.nseg; ++g) {
      const int64_t lo = a.bounds[g], hi = a.bounds[g + 1];
      if (lo >= rows) break;
      const int64_t L = min(hi, rows) - lo;
      const int64_t p = (int64_t)a.P[g * a.pitch + k];
      if (p == L) {  // the whole segment is one run: keep it open
        open += L;
        continue;
      }
      const int64_t x = open + p;
      if (mode == kFoldStripe && pstr < 0) {
        pstr = x;
      } else if (x > 0) {
        atomicAdd(&a.hist[kDiag * (n + 1) + x], wgt);
      }
      open = (hi <= rows) ? (int64_t)a.S[g * a.pitch + k] : 0;
    }
    if (mode == kFoldFinal) {
      if (open > 0) atomicAdd(&a.hist[kDiag * (n + 1) + open], wgt);
    } else {
      const int64_t top = a.bounds[0], bot = a.bounds[a.nseg];
      int64_t sstr = 0;
      if (top >= rows) {
        pstr = 0;                 // diagonal does not reach this stripe
      } else if (pstr < 0) {
        pstr = open;              // stripe is one run (full)
        sstr = open;
      } else if (bot <= rows) {
        sstr = open;              // run open at the stripe's bottom edge
      } else if (open > 0) {      // diagonal ended inside the stripe
        atomicAdd(&a.hist[kDiag * (n + 1) + open], wgt);
      }
      a.out_p[k] = (int32_t)pstr;
      a.out_s[k] = (int32_t)sstr;
    }
  }
}

}  // namespace rqa
