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

#include "rqa_runs.cuh"

namespace rqa {

enum FoldMode : int { kFoldFinal = 0, kFoldStripe = 1 };

struct SymFoldArgs {
  // band level (compact layout, see band_offset)
  const uint16_t* P;
  const uint16_t* S;
  const uint32_t* colsum;
  int64_t row_lo, row_hi, H;
  int nb;
  // stripe level (final cross-stripe fold): nseg stripes, pitch n
  const int32_t* sp;          // [nseg][n] diagonal prefix
  const int32_t* ss;          // [nseg][n] diagonal suffix
  const uint2* scol;          // [nseg][n] column-part summary (first=top, last=bottom)
  const int64_t* bounds;      // nseg+1 stripe rows (device)
  int nseg;
  const uint32_t* rowlead;    // [n]
  int64_t n;
  unsigned long long* hist;   // [3][n+1]
  int32_t* out_p;             // stripe mode outputs
  int32_t* out_s;
  uint2* out_col;
};

// Segments whose loads a fold thread issues together.
constexpr int kFoldBatch = 8;

// Block-local line histogram of the fold kernels: shared 32-bit bins for
// lengths < kFoldBins (runs that cross segment edges are plentiful, e.g. one
// white run per hook and band), flushed once per block; longer runs go to
// 64-bit global atomics.  Wider than the band kernel's bins: junction runs of
// smooth data are often longer than a band, and global atomics on a few hot
// lengths serialise in L2.
#ifndef RQA_FOLD_BINS
#define RQA_FOLD_BINS 4096
#endif
constexpr int kFoldBins = RQA_FOLD_BINS;

struct FoldHist {
  uint32_t sh;               // shared-window address of [3][kFoldBins] u32 bins
  unsigned long long* g;     // [3][n+1]
  int64_t stride;            // n+1
  __device__ __forceinline__ void add(int kind, int64_t len, uint32_t w) const {
    if (len < kFoldBins) {
      const uint32_t addr = sh + 4u * (uint32_t)(kind * kFoldBins + (int)len);
      asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(w) : "memory");
    } else {
      atomicAdd(&g[kind * stride + len], (unsigned long long)w);
    }
  }
};

struct FoldBins {
  uint32_t* sh;
  __device__ __forceinline__ void init() {
    for (int q = threadIdx.x; q < 3 * kFoldBins; q += blockDim.x) sh[q] = 0u;
    __syncthreads();
  }
  __device__ __forceinline__ void flush(unsigned long long* g, int64_t n) {
    __syncthreads();
    for (int q = threadIdx.x; q < 3 * kFoldBins; q += blockDim.x) {
      const uint32_t c = sh[q];
      if (c) atomicAdd(&g[(q / kFoldBins) * (n + 1) + (q % kFoldBins)], (unsigned long long)c);
    }
  }
};

__host__ __device__ __forceinline__ int64_t sym_band_offset(int64_t b, int64_t n, int64_t row_lo,
                                                            int64_t H) {
  return b * (n - row_lo) - H * (b * (b - 1) / 2);
}

// Diagonal k >= 0 folded over the segments (height H) of [row_lo, row_hi);
// mode: kFoldFinal counts every run, kFoldStripe reports the runs touching
// the stripe's top / bottom edges.  Offsets advance incrementally (compact layout).
// Body of the diagonal fold for block `bid` of `nblk` (the fused fold kernel
// runs it next to the hook fold; bins: the block's shared histogram).
__device__ __forceinline__ void fold_diag_body(const SymFoldArgs& a, const int mode, int64_t bid,
                                               int64_t nblk, uint32_t* bins) {
  const int64_t n = a.n;
  FoldBins fb{bins};
  fb.init();
  const FoldHist h{smem_u32(bins), a.hist, n + 1};
  // a thread folds diagonals t and n-1-t: their segment counts add up to
  // about the same for every thread (the upper triangle is balanced)
  for (int64_t t = bid * (int64_t)blockDim.x + threadIdx.x; t < (n + 1) / 2;
       t += nblk * blockDim.x)
  for (int side = 0; side < 2; ++side) {
    const int64_t k = side ? n - 1 - t : t;
    if (side && k == t) break;
    const unsigned long long wgt = (k == 0) ? 1ull : 2ull;
    const int64_t rows = n - k;
    int64_t open = 0, pstr = -1;
    int64_t lo = a.row_lo, off = k, stride = n - a.row_lo;
    const int64_t nseg_k = min((int64_t)a.nb, (rows - a.row_lo + a.H - 1) / a.H);
    // segments in batches: all loads of a batch are issued before the
    // (sequential) monoid walk (prefetching the next batch measured slower here)
    for (int64_t g0 = 0; g0 < nseg_k; g0 += kFoldBatch) {
      uint16_t pv[kFoldBatch], sv[kFoldBatch];
#pragma unroll
      for (int q = 0; q < kFoldBatch; ++q) {
        const int64_t oq = off + q * stride - a.H * (int64_t)(q * (q - 1) / 2);
        const bool in = g0 + q < nseg_k;
        pv[q] = in ? a.P[oq] : (uint16_t)0;
        sv[q] = in ? a.S[oq] : (uint16_t)0;
      }
#pragma unroll
      for (int q = 0; q < kFoldBatch; ++q) {
        if (g0 + q < nseg_k) {
          const int64_t hi = min(lo + a.H, a.row_hi);
          const int64_t L = min(hi, rows) - lo;
          const int64_t p = (int64_t)pv[q];
          if (p == L) {
            open += L;
          } else {
            const int64_t x = open + p;
            if (mode == kFoldStripe && pstr < 0) pstr = x;
            else if (x > 0) h.add(kDiag, x, (uint32_t)wgt);
            open = (hi <= rows) ? (int64_t)sv[q] : 0;
          }
          lo += a.H;
        }
      }
      off += kFoldBatch * stride - a.H * (int64_t)(kFoldBatch * (kFoldBatch - 1) / 2);
      stride -= kFoldBatch * a.H;
    }
    if (mode == kFoldFinal) {
      if (open > 0) h.add(kDiag, open, (uint32_t)wgt);
    } else {
      int64_t sstr = 0;
      if (a.row_lo >= rows) {
        pstr = 0;
      } else if (pstr < 0) {
        pstr = open;
        sstr = open;
      } else if (a.row_hi <= rows) {
        sstr = open;
      } else if (open > 0) {
        h.add(kDiag, open, (uint32_t)wgt);
      }
      a.out_p[k] = (int32_t)pstr;
      a.out_s[k] = (int32_t)sstr;
    }
  }
  fb.flush(a.hist, n);
}

__global__ void __launch_bounds__(256, 4) sym_fold_diag(const SymFoldArgs a, const int mode) {
  __shared__ uint32_t bins[3 * kFoldBins];
  fold_diag_body(a, mode, blockIdx.x, gridDim.x, bins);
}

}  // namespace rqa

// ===========================================================================
// Folds of the work-unit kernel (rqa_unit.cuh).  Diagonals use sym_fold_diag
// with per-band segments (after fix_diag_pieces); hooks combine the per-band
// column parts with the per-unit row pieces of the row's own band.
// ===========================================================================
namespace rqa {

struct UnitFoldArgs {
  const uint32_t* colsum;      // compact per band (height H)
  const uint2* rowpiece;       // [nunits][H]
  const int4* units_by_band;   // (band, xa, xb, idx) sorted by band then xa
  const int32_t* band_start;   // [nb+1] into units_by_band
  int64_t row_lo, row_hi, H, HS, D;
  int nb;
  int64_t n;
  unsigned long long* hist;
  uint2* out_col;              // stripe mode: column part per c
  uint2* out_row;              // stripe mode: row part per row (rows of the stripe)
};

__device__ __forceinline__ void fold_hooks_body(const UnitFoldArgs& a, const int mode,
                                                int64_t bid, int64_t nblk, uint32_t* bins) {
  const int64_t n = a.n;
  FoldBins fb{bins};
  fb.init();
  const FoldHist h{smem_u32(bins), a.hist, n + 1};
  // a thread folds hooks t and n-1-t (balanced band counts, as sym_fold_diag)
  for (int64_t t = bid * (int64_t)blockDim.x + threadIdx.x; t < (n + 1) / 2;
       t += nblk * blockDim.x)
  for (int side = 0; side < 2; ++side) {
    const int64_t c = side ? n - 1 - t : t;
    if (side && c == t) break;
    // column part: bands above row c
    Seg acc{0u, 0u, 0u};
    {
      int64_t lo = a.row_lo, off = c - a.row_lo, stride = n - a.row_lo;
      const int64_t nbc = c > a.row_lo ? min((int64_t)a.nb, (c - a.row_lo + a.H - 1) / a.H) : 0;
      // batch g is consumed while batch g+1 is loading (the fold is bound by
      // load latency: one dependent monoid step per band)
      uint32_t vn[kFoldBatch];
      auto load = [&](int64_t g0) {
#pragma unroll
        for (int q = 0; q < kFoldBatch; ++q) {
          // next band: offset grows by (n - lo_g), index shrinks by H
          const int64_t oq = off + q * (stride - a.H) - a.H * (int64_t)(q * (q - 1) / 2);
          vn[q] = g0 + q < nbc ? __ldg(a.colsum + oq) : 0u;
        }
        off += kFoldBatch * (stride - a.H) - a.H * (int64_t)(kFoldBatch * (kFoldBatch - 1) / 2);
        stride -= kFoldBatch * a.H;
      };
      if (nbc > 0) load(0);
      for (int64_t g0 = 0; g0 < nbc; g0 += kFoldBatch) {
        uint32_t vv[kFoldBatch];
#pragma unroll
        for (int q = 0; q < kFoldBatch; ++q) vv[q] = vn[q];
        if (g0 + kFoldBatch < nbc) load(g0 + kFoldBatch);
#pragma unroll
        for (int q = 0; q < kFoldBatch; ++q) {
          if (g0 + q < nbc) {
            const int64_t hi = min(lo + a.H, a.row_hi);
            const int64_t L = min(hi, c) - lo;
            const uint32_t v = vv[q];
            const uint32_t top = v >> 16, bot = v & 0xffffu;
            if ((int64_t)run_len(top) == L && acc.uniform && run_bit(top) == run_bit(acc.first)) {
              acc.first = acc.last = acc.first + (uint32_t)(L << 1);  // uniform + uniform
            } else {
              acc = seg_combine(acc, Seg{top, bot, (int64_t)run_len(top) == L ? 1u : 0u}, h);
            }
            lo += a.H;
          }
        }
      }
    }
    // row part: pieces of row c (only if the row belongs to these bands)
    Seg row{0u, 0u, 0u};
    if (c >= a.row_lo && c < a.row_hi) {
      const int64_t rel = c - a.row_lo;
      const int bc = (int)(rel / a.H);
      const int64_t lr = rel - (int64_t)bc * a.H;
      const int r = (int)(lr / a.HS);
      const int64_t rows = n - c;  // row part: diagonals [0, n-c)
      for (int q = a.band_start[bc]; q < a.band_start[bc + 1]; ++q) {
        const int4 u = a.units_by_band[q];
        const int64_t k0 = max((int64_t)(u.y - r) * a.D, (int64_t)0);
        const int64_t k1 = min((int64_t)(u.z - r) * a.D, rows);
        if (k1 <= k0) continue;
        const uint2 p = a.rowpiece[(int64_t)u.w * a.H + lr];
        row = seg_combine(row, Seg{p.x, p.y, (int64_t)run_len(p.x) == k1 - k0 ? 1u : 0u}, h);
      }
    }
    if (mode == kFoldFinal) {
      seg_flush(seg_combine(acc, row, h), h);
    } else {
      a.out_col[c] = make_uint2(acc.first, acc.last);
      if (c >= a.row_lo && c < a.row_hi) a.out_row[c] = make_uint2(row.first, row.last);
    }
  }
  fb.flush(a.hist, n);
}

__global__ void __launch_bounds__(256, 4) unit_fold_hooks(const UnitFoldArgs a, const int mode) {
  __shared__ uint32_t bins[3 * kFoldBins];
  fold_hooks_body(a, mode, blockIdx.x, gridDim.x, bins);
}

// Both folds in one launch: blocks [0, diag_blocks) fold diagonals, the rest
// fold hooks (independent inputs; the two latency-bound folds overlap).
__global__ void __launch_bounds__(256, 4) unit_fold_all(const SymFoldArgs d, const UnitFoldArgs u,
                                                        const int mode, const int diag_blocks) {
  __shared__ uint32_t bins[3 * kFoldBins];
  if ((int)blockIdx.x < diag_blocks)
    fold_diag_body(d, mode, blockIdx.x, diag_blocks, bins);
  else
    fold_hooks_body(u, mode, blockIdx.x - diag_blocks, gridDim.x - diag_blocks, bins);
}


// Diagonal band segments cut by a work-unit boundary (rqa_unit.cuh): unit u
// walked the upper part (slots 0..rA, open at the cut) and unit u+1 of the
// same band the lower part; join the two halves into the band-level P/S the
// diagonal fold reads, counting the run that meets at the cut (or, for a
// segment cut by the matrix's right edge, the last run).  One thread per
// (unit, rA, lane) record; the geometry decides which records were written.
struct DiagPieceArgs {
  const int4* units_by_band;  // (band, xa, xb, idx) in idx order
  int nunits;
  const uint2* drec;          // [nunits][R-1][D]
  uint16_t* P;                // band-level compact layout (height H)
  uint16_t* S;
  int64_t row_lo, row_hi, n, H, HS, D;
  int R;
  unsigned long long* hist;
  int64_t cap_ps, cap_drec;  // allocated entries (checked build, RQA_CHECKS)
};

__global__ void fix_diag_pieces(const DiagPieceArgs a) {
  const int64_t per = (int64_t)(a.R - 1) * a.D;
  const int64_t total = (int64_t)a.nunits * per;
  const GHist h{a.hist, a.n + 1};
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int u = (int)(q / per);
    const int rA = (int)((q % per) / a.D);
    const int delta = (int)(q % a.D);
    const int4 U = a.units_by_band[u];
    if (u + 1 >= a.nunits || a.units_by_band[u + 1].x != U.x) continue;  // last unit of its band
    const int64_t i0 = a.row_lo + (int64_t)U.x * a.H;
    const int64_t hrows = min(i0 + a.H, a.row_hi) - i0;
    const int64_t nrem = a.n - i0;
    const int64_t kd = (int64_t)(U.z - 1) * a.D - (int64_t)rA * a.HS + delta;
    if (kd < 0 || kd >= nrem) continue;
    const int64_t brows = min(hrows, nrem - kd);
    if (rA >= (brows - 1) / a.HS) continue;  // the segment ended inside unit u
    const uint2 rec = a.drec[q];
    const int64_t LA = (int64_t)(rA + 1) * a.HS, LB = brows - LA;
    const int64_t PA = rec.x & 0xffffu, SA = rec.x >> 16;
    const int64_t PB = rec.y & 0xffffu, SB = (rec.y >> 16) & 0x7fffu;
    const bool open = (rec.y >> 31) == 0u;
    const bool allA = PA == LA, allB = PB == LB;
    const uint32_t w = kd == 0 ? 1u : 2u;
    const int64_t Pv = allA ? LA + PB : PA;
    const int64_t Sv = !open ? 0 : allB ? SA + LB : SB;
    if (!allA && !allB) {
      if (SA + PB > 0) h.add(kDiag, SA + PB, w);  // the run meeting at the cut
    } else if (!open && allB && !allA) {
      h.add(kDiag, SA + LB, w);  // last run, ends at the matrix edge
    }
    const int64_t off = sym_band_offset(U.x, a.n, a.row_lo, a.H) + kd;
    RQA_DCHECK_AT(16, q < a.cap_drec && off >= 0 && off < a.cap_ps);
    a.P[off] = (uint16_t)Pv;
    a.S[off] = (uint16_t)Sv;
  }
}

// Final fold over stripes (multi-GPU) for the work-unit layout.
struct UnitStitchArgs {
  const int32_t* sp;        // [nseg][n] diagonal prefix
  const int32_t* ss;        // [nseg][n] diagonal suffix
  const uint2* scol;        // [nseg][n] column part per stripe
  const uint2* srow;        // [n] row part (each row from its own stripe)
  const int64_t* bounds;    // nseg+1
  int nseg;
  int64_t n;
  unsigned long long* hist;
};

__global__ void __launch_bounds__(256, 4) unit_fold_stripes(const UnitStitchArgs a) {
  const int64_t n = a.n;
  // block-local bins as in the folds (global atomics on a few hot lengths
  // serialise in L2)
  __shared__ uint32_t bins[3 * kFoldBins];
  FoldBins fb{bins};
  fb.init();
  const FoldHist h{smem_u32(bins), a.hist, n + 1};
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    {
      const unsigned long long wgt = (k == 0) ? 1ull : 2ull;
      const int64_t rows = n - k;
      int64_t open = 0;
      for (int g = 0; g < a.nseg; ++g) {
        const int64_t lo = a.bounds[g], hi = a.bounds[g + 1];
        if (lo >= rows) break;
        if (hi <= lo) continue;
        const int64_t L = min(hi, rows) - lo;
        const int64_t p = a.sp[g * n + k];
        if (p == L) {
          open += L;
          continue;
        }
        const int64_t x = open + p;
        if (x > 0) h.add(kDiag, x, (uint32_t)wgt);
        open = (hi <= rows) ? (int64_t)a.ss[g * n + k] : 0;
      }
      if (open > 0) h.add(kDiag, open, (uint32_t)wgt);
    }
    {
      const int64_t c = k;
      Seg acc{0u, 0u, 0u};
      for (int g = 0; g < a.nseg; ++g) {
        const int64_t lo = a.bounds[g], hi = a.bounds[g + 1];
        if (lo >= c) break;
        if (hi <= lo) continue;
        const int64_t L = min(hi, c) - lo;
        const uint2 v = a.scol[g * n + c];
        acc = seg_combine(acc, Seg{v.x, v.y, (int64_t)run_len(v.x) == L ? 1u : 0u}, h);
      }
      const uint2 rp = a.srow[c];
      const Seg row{rp.x, rp.y, (int64_t)run_len(rp.x) == n - c ? 1u : 0u};
      seg_flush(seg_combine(acc, row, h), h);
    }
  }
  fb.flush(a.hist, n);
}

}  // namespace rqa
