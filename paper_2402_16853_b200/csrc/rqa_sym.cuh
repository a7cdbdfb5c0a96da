// rqa_sym.cuh -- upper-triangle band kernel (exact symmetry R = R^T).
//
// Only cells with k = j - i >= 0 are evaluated: half the FP64 work of the
// full matrix.  The lines of the full matrix are recovered exactly:
//   * diagonal lines: diagonal -k is a copy of diagonal k (k > 0 counts 2x);
//   * vertical / white-vertical lines: column c of the full matrix equals the
//     "hook" c = upper column c above the diagonal (rows 0..c-1) followed by
//     upper row c from the diagonal (columns c..n-1), because R(r,c) = R(c,r).
// The hook's row part lives in the band holding row c (row phase); its
// column part is cut into one segment per band (column phase) and stitched
// by fold_hooks (rqa_fold.cuh) with the run monoid of rqa_runs.cuh.
//
// Geometry as in rqa_band.cuh: band of H = R*HS rows, HS = D = 32*NW,
// iteration x covers diagonals kd = x*D - r*HS + delta in slot r, lane
// delta = 32*warp + lane; column of step t is i0 + t + x*D + delta for every
// slot (one shared column load feeds R cells).  Columns are met bottom-up by
// the diagonal sweep, so the column phase consumes them bottom-up.
#pragma once
#include "rqa_band.cuh"
#include "rqa_runs.cuh"

namespace rqa {

struct SymArgs {
  const double* s;           // device samples (zero padded both sides)
  int64_t len, n;
  int64_t row_lo, row_hi;    // rows of this launch; bands start at row_lo
  double thr;
  int64_t theiler;
  int m, tau;
  uint16_t* P;               // compact [band][kd], kd in [0, n - i0): 1-run at band top
  uint16_t* S;               // compact: 1-run at band bottom
  uint32_t* colsum;          // compact [band][c - i0]: (top run len<<1|bit) << 16 ... see pack_col
  uint32_t* rowlead;         // [n]: first run of upper row i from the diagonal
  unsigned long long* hist;  // [3][n+1]
  unsigned long long* points;
  int skip;                  // profiling only (RQA_SKIP): 1 diag runs, 2 row phase, 4 column phase
  int flush_mask;            // shared bins emptied when ((iteration + 1) & flush_mask) == 0
                             // (4095; RQA_FLUSH_EVERY=2^k for tests of that path)
  unsigned long long* timers;  // profiling only (RQA_TIMERS): [4] cycles compute/rows/cols/other
  // f32 filter kernels (PREC = 1, rqa_unit.cuh): float32 evaluation with a
  // certified band around the threshold; words with a cell inside the band
  // are re-evaluated in float64 (and, in fp32 mode, in scalar float32).
  const float* sf;           // device samples rounded to float32, same padding as s
  float c32;                 // band centre: fast-path bit = (acc32 - c32 < 0)
  float band32;              // half-width: |acc32 - c32| <= band32 is ambiguous
  float thr32;               // fp32-mode threshold (T*32 for L2 with m > 1, else fl32(radius))
  int prec_mode;             // 0: exact (ambiguous words take the float64 bits); 1: fp32 mode
  int all_amb;               // 1: every word is re-evaluated (band not certifiable)
  unsigned long long* mism;  // fp32 mode: cells whose fp32 and fp64 decisions differ
  double dstar;              // prefilter (PREC 2): |d| <= dstar for every term of a candidate
  // packed float32 prefilter predicate (PREC 2, m <= 4): a cell is a
  // component candidate iff fma(d32, d32, pre_negd2) < 0 (sign bit), a
  // certified superset of |d| <= dstar (rqa_capi.cu plan_prefilter)
  float pre_negd2;
};

// Compact per-band offset of entries kd (or c - i0) in [0, n - i0).
__host__ __device__ __forceinline__ int64_t band_offset(int64_t b, int64_t n, int64_t row_lo,
                                                        int64_t H) {
  return b * (n - row_lo) - H * (b * (b - 1) / 2);
}

// Column-segment summary: top and bottom runs, 15-bit lengths (H <= 32767).
__host__ __device__ __forceinline__ uint32_t pack_col(uint32_t top, uint32_t bot) {
  return ((top & 0xffffu) << 16) | (bot & 0xffffu);
}

// Capacities (powers of two) of a warp's streaming candidate list (prefilter
// kernels) are per variant (rqa_unit.cuh kCandCapOf): pending entries plus
// one slot word's; a denser word is resolved per lane.

struct SymSmem {
  int H, HS, D, W, CW;
  size_t off_row, off_col0, off_col1, off_rowbuf, off_prev, off_colst, off_rowst, off_queue,
      off_hist, off_cand, off_cres, off_rowf, off_colf0, off_colf1, total;
  int CWF;  // float32 column window (f32pred)
  // esize 8: float64 row/column windows; 4: float32 windows (f32 filter
  // kernels), the row window stored as R/2 interleaved slot pairs of
  // HS + W + 4 float2 each (rqa_unit.cuh, packed f32x2 evaluation).
  // cand_cap: entries of the per-warp streaming candidate list (prefilter kernels)
  // f32pred: float32 copies of the windows for the packed prefilter
  // predicate (row window as R/2 slot pairs of HS + W + 4 float2, two float
  // column buffers), appended at the end
  __host__ __device__ SymSmem(int NW, int R, int W_, int esize = 8, int cand_cap = 0,
                              bool f32pred = false) {
    D = 32 * NW;
    HS = D;
    H = R * HS;
    W = W_;
    off_row = 0;
    if (esize == 8) {
      CW = ((HS + D + W + 2) + 1) & ~1;
      const size_t row_elems = ((size_t)(H + W) + 2) & ~(size_t)1;
      off_col0 = off_row + row_elems * sizeof(double);
    } else {
      CW = ((HS + D + W + 4) + 3) & ~3;  // TMA sizes are multiples of 16 bytes
      const size_t row_bytes = (size_t)(R + 1) * (HS + W + 4) * sizeof(float);
      off_col0 = off_row + ((row_bytes + 15) & ~(size_t)15);
    }
    off_col1 = off_col0 + (size_t)CW * esize;
    off_rowbuf = off_col1 + (size_t)CW * esize;
    off_prev = off_rowbuf + (size_t)NW * H * sizeof(uint32_t);
    off_colst = off_prev + 2 * (size_t)H * sizeof(uint32_t);
    off_rowst = off_colst + (size_t)NW * R * 32 * sizeof(uint2);
    off_queue = (off_rowst + (size_t)R * D * sizeof(uint2) + 15) & ~(size_t)15;  // 16-B events
    off_hist = off_queue + (size_t)NW * kQueueCap * sizeof(uint4);
    // bins, two mbarriers (16 B), the dummy bin of hist_red (16 B reserved)
    off_cand = off_hist + 3 * kSmemBins * sizeof(uint32_t) + 32;
    off_cres = off_cand + (size_t)NW * cand_cap * sizeof(uint16_t);
    total = off_cres;
    CWF = ((HS + D + W + 4) + 3) & ~3;
    off_rowf = off_colf0 = off_colf1 = total;
    if (f32pred) {
      off_rowf = (total + 15) & ~(size_t)15;
      off_colf0 = (off_rowf + (size_t)(R / 2) * (HS + W + 4) * sizeof(float2) + 15) & ~(size_t)15;
      off_colf1 = off_colf0 + (size_t)CWF * sizeof(float);
      total = off_colf1 + (size_t)CWF * sizeof(float);
    }
  }
};

// Set bit T of dw iff acc <= thr: DSETP + predicated LOP3 (no SEL chains).
__device__ __forceinline__ void setbit_le(uint32_t& dw, double acc, double thr, uint32_t bit) {
  asm("{\n\t.reg .pred p;\n\tsetp.le.f64 p, %1, %2;\n\t@p or.b32 %0, %0, %3;\n\t}"
      : "+r"(dw)
      : "d"(acc), "d"(thr), "r"(bit));
}

// A piece of a diagonal ends: returns P | S << 16, P = its top run (length if
// it is a run of ones, else 0) and, if the piece ends at the band's bottom
// edge or at a work-unit boundary (open), S = its bottom run; a piece cut by
// the matrix's right edge (closed) counts its last run here and reports S = 0.
__device__ __forceinline__ uint32_t diag_piece_end(const RunState& st, bool open,
                                                   const LineSink& sink) {
  const Seg g = runs_finish(st);
  const uint32_t p = run_bit(g.first) ? run_len(g.first) : 0u;
  uint32_t s = 0u;
  if (open) {
    s = run_bit(g.last) ? run_len(g.last) : 0u;
  } else if (!g.uniform) {
    sink(g.last);
  }
  return p | (s << 16);
}

}  // namespace rqa
