// rqa_device.cuh -- device-side building blocks of the B200 RQA engine.
//
// Bit conventions used everywhere in this file:
//   * a "diagonal word" is held by one lane: bit t is the cell at step t of a
//     32-step chunk, i.e. row (chunk_row0 + t) of the lane's diagonal;
//   * a "row word" (after transpose32) is held by lane t: bit l is the cell of
//     row (chunk_row0 + t) at column (column_base + l), LSB = leftmost column.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace rqa {

enum Metric : int { kL1 = 0, kL2 = 1, kLinf = 2 };
enum HistKind : int { kDiag = 0, kVert = 1, kWhite = 2 };

// Shared-memory histogram bins per kind; longer lines go to global memory.
constexpr int kSmemBins = 1024;

struct BandArgs {
  const double* s;          // device samples, s[-pad .. len+pad) readable (zero padded)
  int64_t len;              // number of samples
  int64_t n;                // number of embedded vectors
  int64_t row_lo, row_hi;   // rows covered by this launch: bands [row_lo + b*H, ...)
  double thr;               // T* for L2 with m>1 (sqrt removed exactly), radius otherwise
  int64_t theiler;          // cells with |i-j| < theiler are forced to 0
  int m, tau;               // runtime embedding (direct mode only)
  uint16_t* P;              // [nbands][n] prefix run at band top, per diagonal k >= 0
  uint16_t* S;              // [nbands][n] suffix run at band bottom
  unsigned long long* hist; // [3][n+1]: diagonal, vertical, white vertical
  unsigned long long* points;
};

// 32x32 bit transpose across a warp (lane l word bit t -> lane t word bit l).
__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
#pragma unroll
  for (int j = 16; j >= 1; j >>= 1) {
    const uint32_t m = (j == 16) ? 0x0000FFFFu
                     : (j == 8)  ? 0x00FF00FFu
                     : (j == 4)  ? 0x0F0F0F0Fu
                     : (j == 2)  ? 0x33333333u
                                 : 0x55555555u;
    const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
    x = (lane & j) ? ((x & ~m) | ((y >> j) & m)) : ((x & m) | ((y << j) & ~m));
  }
  return x;
}

// Per-lane constants of the rotate-and-select 32x32 bit transpose: stage j
// exchanges j-blocks with lane^j; the partner word is rotated left by j (or
// 32-j when lane bit j is set) and bit-selected into place with mask M_j.
struct Transposer {
  uint32_t M[5];
  uint32_t amt[5];
  __device__ __forceinline__ explicit Transposer(int lane) {
#pragma unroll
    for (int s = 0; s < 5; ++s) {
      const int j = 16 >> s;
      const uint32_t m = (j == 16) ? 0x0000FFFFu
                       : (j == 8)  ? 0x00FF00FFu
                       : (j == 4)  ? 0x0F0F0F0Fu
                       : (j == 2)  ? 0x33333333u
                                   : 0x55555555u;
      const bool hi = (lane & j) != 0;
      M[s] = hi ? m : ~m;
      amt[s] = hi ? (uint32_t)(32 - j) : (uint32_t)j;
    }
  }
  // lane l word bit t -> lane t word bit l
  __device__ __forceinline__ uint32_t operator()(uint32_t x) const {
#pragma unroll
    for (int s = 0; s < 5; ++s) {
      const int j = 16 >> s;
      const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
      const uint32_t r = (j == 16) ? __funnelshift_l(y, y, 16) : __funnelshift_l(y, y, amt[s]);
      uint32_t o;  // bit select (x & ~M) | (r & M) in one LOP3
      asm("lop3.b32 %0, %1, %2, %3, 0xD8;" : "=r"(o) : "r"(x), "r"(r), "r"(M[s]));
      x = o;
    }
    return x;
  }
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// 32-bit shared-window load (keeps the window base out of the address math).
// volatile: never moved across barriers; no memory clobber, so it does not
// pin the surrounding loads and stores.
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }

__device__ __forceinline__ uint32_t low_mask(int bits) {
  return bits >= 32 ? 0xffffffffu : ((1u << bits) - 1u);
}

// Line-length histograms of one CTA: 32-bit shared-memory bins for lengths
// < kSmemBins (red.shared, no generic addressing), 64-bit global atomics
// beyond.  kind: kDiag, kVert, kWhite.
struct Hist {
  uint32_t sh;               // shared-window address of [3][kSmemBins] u32 bins
  unsigned long long* g;     // [3][n+1]
  int64_t stride;            // n+1
  __device__ __forceinline__ void add(int kind, int64_t len, uint32_t w) const {
    if (len < kSmemBins) {
      const uint32_t addr = sh + 4u * (uint32_t)(kind * kSmemBins + (int)len);
      asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(w) : "memory");
    } else {
      atomicAdd(&g[kind * stride + len], (unsigned long long)w);
    }
  }
};

// Global-only histogram (fold kernels).
struct GHist {
  unsigned long long* g;
  int64_t stride;
  __device__ __forceinline__ void add(int kind, int64_t len, uint32_t w) const {
    atomicAdd(&g[kind * stride + len], (unsigned long long)w);
  }
};

// Open diagonal 1-run of one lane slot.  `rooted` marks a run that started at
// the band's top edge: it is not counted here but reported as the band's
// prefix P[k] for the fold kernel (engine.py:287-319 carry contract, restated
// as a segment monoid).
struct DiagRun {
  int32_t len;
  int32_t rooted;
};

__device__ __forceinline__ void diag_end_run(DiagRun& st, uint16_t* Pk, uint32_t weight,
                                             const Hist& h) {
  if (st.rooted) {
    *Pk = (uint16_t)st.len;
    st.rooted = 0;
  } else if (st.len > 0) {
    h.add(kDiag, st.len, weight);
  }
  st.len = 0;
}

// Consume the first `lc` bits of diagonal word x; if lc < l the diagonal hit
// the matrix's right edge inside the band, which closes the open run.
__device__ __forceinline__ void diag_word(uint32_t x, int lc, int l, DiagRun& st,
                                          uint16_t* Pk, uint32_t weight, const Hist& h) {
  if (lc > 0) {
    const uint32_t full = low_mask(lc);
    x &= full;
    if (x == full) {
      st.len += lc;
    } else if (x == 0u) {
      if (st.len | st.rooted) diag_end_run(st, Pk, weight, h);
    } else {
      const int a = __ffs(~x) - 1;  // leading ones (continue the open run)
      st.len += a;
      diag_end_run(st, Pk, weight, h);
      uint32_t y = (a >= 31) ? 0u : (x & ~((2u << a) - 1u));
      while (y) {
        const int s0 = __ffs(y) - 1;
        const uint32_t zeros = ~y & (0xffffffffu << s0) & full;
        if (zeros == 0u) {  // run reaches the end of the consumed bits: stays open
          st.len = lc - s0;
          break;
        }
        const int e = __ffs(zeros) - 1;
        h.add(kDiag, e - s0, weight);
        y &= (e >= 32) ? 0u : (0xffffffffu << e);
      }
    }
  }
  if (lc < l && (st.len | st.rooted)) diag_end_run(st, Pk, weight, h);
}

// Open row run: `bit` is the value of the open run (-1 before the first
// valid column), `len` its length.  Row runs of ones are vertical lines and
// runs of zeroes white vertical lines, by the exact symmetry R = R^T.
struct RowRun {
  int32_t bit;
  int32_t len;
};

__device__ __forceinline__ void row_emit(const RowRun& st, const Hist& h) {
  if (st.len > 0) h.add(st.bit ? kVert : kWhite, st.len, 1u);
}

// Consume `nb` (1..32) bits of x (bit 0 first) into the open row run.
__device__ __forceinline__ void row_bits(uint32_t x, int nb, RowRun& st, const Hist& h) {
  const uint32_t full = low_mask(nb);
  x &= full;
  if (st.bit < 0) {
    st.bit = (int)(x & 1u);
    st.len = 0;
  }
  const uint32_t same = st.bit ? x : (~x & full);  // bits equal to the open run's value
  if (same == full) {
    st.len += nb;
    return;
  }
  int pos = 0;
  while (pos < nb) {
    uint32_t diff = (st.bit ? ~x : x) & full;       // bits that differ from the open run
    diff = (pos >= 32) ? 0u : (diff >> pos);
    if (diff == 0u) {
      st.len += nb - pos;
      return;
    }
    const int run = __ffs(diff) - 1;
    st.len += run;
    row_emit(st, h);
    st.bit ^= 1;
    st.len = 0;
    pos += run;
  }
}

}  // namespace rqa
