// rqa_unit.cuh -- upper-triangle kernel over 2-D work units.
//
// A work unit is (band b, iteration range [x_a, x_b)) of the diagonal sweep
// of the upper-triangle band kernel: bands of H = R*HS rows are cut along the sweep
// so that every CTA gets a bounded amount of work, which balances the SMs
// for any n and lets a GPU's share of a multi-GPU run be spread over all of
// its SMs.  What crosses a unit boundary is stitched by the folds:
//   * diagonals: diagonal kd meets slot r of a band at iteration kd/D + r, in
//     the same lane, so its run state is handed from slot r to slot r+1 in
//     registers and the whole band segment is one piece (P/S per band,
//     compact layout with height H).  A work-unit boundary cuts the pieces
//     of at most R-1 slots per lane; both halves go to a record and
//     fix_diag_pieces (rqa_fold.cuh) joins them (units span >= R iterations);
//   * row parts of hooks: each unit reports the first and last run of the
//     piece of the row it covers (rowpiece[unit][row]);
//   * column parts of hooks: a column's slot segment spans iterations x-1 and
//     x; a unit recomputes iteration x_a-1 (cells and row words only) to own
//     the lower parts of the columns it finishes, and leaves the columns that
//     finish at x_b to the next unit.
// Lane delta of warp v walks diagonal kd = x*D - r*HS + 32v + lane of slot r;
// the four slots of a lane share the column of every step.
#pragma once
#include <type_traits>

#include "rqa_sym.cuh"

namespace rqa {

// One work unit: band, first and last+1 iteration, row-piece slot index.
struct Unit {
  int32_t band, xa, xb, idx;
};

struct UnitArgs {
  SymArgs base;            // s, n, row range, thr, theiler, m, tau, P, S, colsum, hist, points
  const Unit* units;       // [nunits], ordered largest work first
  uint2* rowpiece;         // [nunits][H]: (first, last) run of each row's piece
  uint2* drec;             // [nunits][R-1][D]: diagonal pieces cut at the unit's end
                           // (x: upper half P | S << 16, y: lower half P | S << 16 | closed << 31)
  // allocated entries (bounds of the checked build, RQA_CHECKS)
  int64_t cap_ps, cap_cs, cap_drec, cap_piece;
};

// ---------------------------------------------------------------------------
// f32 filter (PREC = 1).  Cells are evaluated in float32 (packed f32x2 over
// slot pairs for the L1/L2 term-reuse kernels); the bit of a cell is the sign
// of acc32 - c32.  The host certifies a band |acc32 - c32| <= band32 outside
// which the float32 decision equals the float64 one (rqa_capi.cu,
// f32_band); a word with a cell inside the band is re-evaluated here, in
// float64 with the reference's operation order (and in scalar float32 with
// the fp32-mode semantics, for the mismatch count).
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long f2_add(unsigned long long x, unsigned long long y) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(x), "l"(y));
  return d;
}
__device__ __forceinline__ unsigned long long f2_mul(unsigned long long x, unsigned long long y) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(x), "l"(y));
  return d;
}
__device__ __forceinline__ unsigned long long f2_pack(float lo, float hi) {
  return ((unsigned long long)__float_as_uint(hi) << 32) | __float_as_uint(lo);
}
__device__ __forceinline__ float f2_lo(unsigned long long x) { return __uint_as_float((uint32_t)x); }
__device__ __forceinline__ float f2_hi(unsigned long long x) {
  return __uint_as_float((uint32_t)(x >> 32));
}

// Re-evaluate the 32 cells (row0 + t, row0 + t + kd), t = 0..31, of one word:
// x = float64 bits (reference semantics, threshold a.thr), y = float32 bits
// (fp32-mode semantics: samples, ufuncs and threshold in float32).
template <int METRIC>
__device__ __forceinline__ uint2 f32_recheck(const SymArgs& a, int64_t row0, int64_t kd) {
  const int m = a.m, tau = a.tau;
  const bool per_comp = (METRIC == kLinf) || m == 1;
  uint32_t w64 = 0u, w32 = 0u;
  for (int t = 0; t < 32; ++t) {
    const int64_t i = row0 + t, j = i + kd;
    bool h64 = true, h32 = true;
    double acc = 0.0;
    float acc32 = 0.0f;
    for (int k = 0; k < m; ++k) {
      const int64_t o = (int64_t)k * tau;
      const double d = __dsub_rn(a.s[i + o], a.s[j + o]);
      const float d32 = __fsub_rn(a.sf[i + o], a.sf[j + o]);
      if (per_comp) {
        h64 &= fabs(d) <= a.thr;
        h32 &= fabsf(d32) <= a.thr32;
      } else {
        const double tm = (METRIC == kL2) ? __dmul_rn(d, d) : fabs(d);
        const float tm32 = (METRIC == kL2) ? __fmul_rn(d32, d32) : fabsf(d32);
        acc = (k == 0) ? tm : __dadd_rn(acc, tm);
        acc32 = (k == 0) ? tm32 : __fadd_rn(acc32, tm32);
      }
    }
    if (!per_comp) {
      h64 = acc <= a.thr;
      h32 = acc32 <= a.thr32;
    }
    w64 |= (h64 ? 1u : 0u) << t;
    w32 |= (h32 ? 1u : 0u) << t;
  }
  return make_uint2(w64, w32);
}

// Prefilter kernels (PREC 2) resolve their candidates warp-cooperatively from
// a per-warp list that streams across the chunks of an iteration: every
// round takes 32 entries at full SIMD width (rqa_unit.cuh, phase 1).  Short
// sums list candidate words (at most R * 32 new entries per chunk, 256
// entries); long sums (m >= 5) list cells, appended per slot word, 512
// entries (two CTAs per SM still fit).
template <int PREC, int M>
#ifndef RQA_CAND_CAP_LONG
#define RQA_CAND_CAP_LONG 512
#endif
constexpr int kCandCapOf = (PREC != 2) ? 0 : (M <= 4 ? 256 : RQA_CAND_CAP_LONG);
// Short-window prefilter kernels evaluate the per-component predicate in
// packed float32 (sub/fma.rn.f32x2 over slot pairs, the sign bit of
// d32*d32 - D32^2 funnel-shifted into the word): 2.5 instructions per cell
// instead of DADD + DSETP + LOP.  It is a certified superset of the float64
// predicate |d| <= D* (rqa_capi.cu plan_prefilter), and every candidate is
// still decided by the exact float64 sum, so the result is unchanged.
template <int PREC, int M, int R>
constexpr bool kF32Pred = (PREC == 2) && (M >= 2) && (M <= 4) && (R % 2 == 0);

template <int METRIC, int M, int TAU, int NW, int R, int MINB, int PREC = 0>
__global__ void __launch_bounds__(NW * 32, MINB)
unit_kernel(const UnitArgs ua, const int W_rt) {
  const SymArgs& a = ua.base;
  constexpr int D = 32 * NW;
  constexpr int HS = D;
  constexpr int H = R * HS;
  constexpr bool kDirect = (M == 0);
  constexpr int kW = kDirect ? 0 : (M - 1) * TAU;
  constexpr bool kLinfAnd = (METRIC == kLinf) && (M >= 2);
  // PREC 2: sparse prefilter for L1/L2 (exact).  Every term of a sum of
  // non-negative terms is <= the float64 sum, so acc <= T implies
  // |d_k| <= D* for every k (D* = max{x : fl(x*x) <= T} for L2, T for L1):
  // the AND of the m shifted per-cell predicates |d| <= D* (as for L-inf)
  // marks the only cells that can be recurrent, and only those are summed.
  constexpr bool kPre = (PREC == 2) && (M >= 2) && (METRIC != kLinf);
  constexpr bool kAnd = kLinfAnd || kPre;
#ifndef RQA_RANGE_END
#define RQA_RANGE_END 0  // A/B: 1 = range test of the segment end in every kernel
#endif
  constexpr bool kRangeEnd = kPre || kLinfAnd || RQA_RANGE_END;  // diagonal pieces, below
  constexpr bool kSquare = (METRIC == kL2) && (M >= 2);
  constexpr int NCH = HS / 32;  // == NW
  static_assert(kAnd ? kW <= 96 : kW <= 48, "term window too large");
  // predicate window of the AND kernels: 32 steps + kW look-ahead bits
  constexpr int NPH = 1 + (kW + 31) / 32;
  static_assert(PREC != 2 || kPre, "prefilter: L1/L2 term-reuse kernels only");
  constexpr bool kF32 = (PREC == 1);
  // packed f32x2 evaluation over slot pairs (2r, 2r+1): L1/L2 term reuse
  constexpr bool kPacked = kF32 && !kDirect && !kLinfAnd && M >= 2 && (R % 2 == 0);
  static_assert(!kF32 || kDirect || kPacked, "f32 filter: packed reuse or direct kernels");
  using F = typename std::conditional<kF32, float, double>::type;
  constexpr int RP = (R + 1) / 2;  // slot pairs
  const int W = kDirect ? W_rt : kW;
  constexpr bool kFP = kF32Pred<PREC, M, R>;
  // Long-window prefilter kernels test consecutive component PAIRS:
  // fl(term_{k-1} + term_k) <= T for k = 1..m-1.  The reference's sum adds
  // non-negative terms in k order and float64 addition is monotone, so its
  // result is >= fl(term_{k-1} + term_k) for every k: the pair predicate is an
  // exact superset of acc <= T (no margin) and about 3x more selective than
  // the per-component one on C4 (2.4 % vs 7.1 % of the cells).
  constexpr bool kPair = kPre && !kFP;
  constexpr int kCandCap = kCandCapOf<PREC, M>;
  const SymSmem L(NW, R, W, (int)sizeof(F), kCandCap, kFP);
  const int PS = HS + W + 4;       // packed row window: float2 elements per slot pair

  extern __shared__ __align__(128) unsigned char smem[];
  F* s_row = reinterpret_cast<F*>(smem + L.off_row);
  float2* s_row2 = reinterpret_cast<float2*>(smem + L.off_row);
  uint32_t* rowbuf = reinterpret_cast<uint32_t*>(smem + L.off_rowbuf);
  uint32_t* prevbuf = reinterpret_cast<uint32_t*>(smem + L.off_prev);
  uint2* colst = reinterpret_cast<uint2*>(smem + L.off_colst);
  uint2* rowst = reinterpret_cast<uint2*>(smem + L.off_rowst);
  uint32_t* sh_hist = reinterpret_cast<uint32_t*>(smem + L.off_hist);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L.off_hist + 3 * kSmemBins * sizeof(uint32_t));

  const Unit unit = ua.units[blockIdx.x];
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int wv = tid >> 5;
  const int delta = 32 * wv + lane;
  const int64_t n = a.n;
  const int64_t b = unit.band;
  const int64_t i0 = a.row_lo + b * H;
  const int64_t i_end = min(i0 + (int64_t)H, a.row_hi);
  const int nrem = (int)(n - i0);
  const int hrows = (int)(i_end - i0);
  const int theiler = (int)min(a.theiler, (int64_t)1 << 30);
  const double thr = a.thr;
  const double athr = kPre ? a.dstar : thr;  // per-component predicate threshold
  // exact float64 sum of one prefilter candidate, in the reference's order
  auto pre_exact = [&](const F* rp, const F* cp) {
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < (M > 0 ? M : 1); ++k) {
      const double d = __dsub_rn((double)rp[k * TAU], (double)cp[k * TAU]);
      const double term = kSquare ? __dmul_rn(d, d) : fabs(d);
      acc = (k == 0) ? term : __dadd_rn(acc, term);
    }
    return acc <= thr;
  };
  const int xa = unit.xa, xb = unit.xb;
  const int xfirst = xa > 0 ? xa - 1 : 0;  // xa-1: recomputed for the columns finishing at xa
  uint32_t* Cb = a.colsum + band_offset(b, n, a.row_lo, H);
  uint2* piece = ua.rowpiece + (int64_t)unit.idx * H;
  const Hist hist{smem_u32(sh_hist), a.hist, n + 1};
  const Transposer tr(lane);
  // this lane's row-word slot (warp wv, row lane of chunk 0, slot 0) as a
  // 32-bit shared address kept in a register; profiling mask likewise
  uint32_t rowbuf_sa = smem_u32(rowbuf + wv * H + lane);
  int skip = a.skip;
  asm volatile("" : "+r"(rowbuf_sa), "+r"(skip));
  EventQueue evq{reinterpret_cast<uint4*>(smem + L.off_queue) + wv * kQueueCap, 0u, 0u,
                 (1u << lane) - 1u};
  evq.ring_sa = smem_u32(evq.ring);
  uint16_t* Pb = a.P + band_offset(b, n, a.row_lo, H);  // band-level diagonal summaries
  uint16_t* Sb = a.S + band_offset(b, n, a.row_lo, H);

  const F* gs;  // samples the windows are staged from
  if constexpr (kF32) gs = a.sf; else gs = a.s;
  for (int q = tid; q < 3 * kSmemBins; q += NW * 32) sh_hist[q] = 0u;
  if constexpr (kPacked) {
    for (int q = tid; q < RP * (HS + W); q += NW * 32) {
      const int pr = q / (HS + W), u = q - pr * (HS + W);
      s_row2[pr * PS + u] = make_float2(gs[i0 + 2 * pr * HS + u], gs[i0 + (2 * pr + 1) * HS + u]);
    }
  } else {
    for (int q = tid; q < H + W; q += NW * 32) s_row[q] = gs[i0 + q];
  }
  if constexpr (kFP) {
    float2* rowf = reinterpret_cast<float2*>(smem + L.off_rowf);
    for (int q = tid; q < (R / 2) * (HS + W); q += NW * 32) {
      const int pr = q / (HS + W), u = q - pr * (HS + W);
      rowf[pr * (HS + W + 4) + u] = make_float2(a.sf[i0 + 2 * pr * HS + u], a.sf[i0 + (2 * pr + 1) * HS + u]);
    }
  }
  for (int q = tid; q < 2 * H; q += NW * 32) prevbuf[q] = 0u;
  for (int q = tid; q < NW * R * 32; q += NW * 32) colst[q] = make_uint2(0u, 0u);
  for (int q = tid; q < R * D; q += NW * 32) rowst[q] = make_uint2(0u, 0u);
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t col_bytes = (uint32_t)(L.CW * sizeof(F));
  const uint32_t colf_bytes = kFP ? (uint32_t)(L.CWF * sizeof(float)) : 0u;
  if (tid == 0) {
    const F* src;
    col_window_src(gs, i0 + (int64_t)xfirst * D, &src);
    mbar_expect_tx_arrive(&bar[0], col_bytes + colf_bytes);
    tma_load_1d(smem + L.off_col0, src, col_bytes, &bar[0]);
    if constexpr (kFP) {
      const float* srcf;
      col_window_src(a.sf, i0 + (int64_t)xfirst * D, &srcf);
      tma_load_1d(smem + L.off_colf0, srcf, colf_bytes, &bar[0]);
    }
  }

  RunState st[R];  // diagonal run state of the current (band, slot) segment
  double win[R][kW > 0 ? kW : 1];
  unsigned long long win2[RP][kW > 0 ? kW : 1];  // packed f32 term windows (kPacked)
  unsigned long long mism = 0;                   // fp32 mode: mismatched cells
  uint32_t ph[R][NPH];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    st[r] = RunState{0u, 0u};
#pragma unroll
    for (int q = 0; q < NPH; ++q) ph[r][q] = 0u;
  }
  uint32_t pts = 0;
  unsigned long long pts64 = 0;

  for (int x = xfirst; x < xb; ++x) {
    const int kx = x * D;
    const int it = x - xfirst;           // local iteration counter (buffer parity)
    const int buf = it & 1;
    const bool warm = x < xa;             // column lower parts only
    if (tid == 0 && x + 1 < xb) {
      const F* src;
      col_window_src(gs, i0 + kx + D, &src);
      mbar_expect_tx_arrive(&bar[buf ^ 1], col_bytes + colf_bytes);
      tma_load_1d(smem + (buf ? L.off_col0 : L.off_col1), src, col_bytes, &bar[buf ^ 1]);
      if constexpr (kFP) {
        const float* srcf;
        col_window_src(a.sf, i0 + kx + D, &srcf);
        tma_load_1d(smem + (buf ? L.off_colf0 : L.off_colf1), srcf, colf_bytes, &bar[buf ^ 1]);
      }
    }
    mbar_wait(&bar[buf], (uint32_t)((it >> 1) & 1));
    const int co = (int)((((uintptr_t)(gs + i0 + kx)) & 15u) / sizeof(F));
    const F* s_col =
        reinterpret_cast<const F*>(smem + (buf ? L.off_col1 : L.off_col0)) + co + delta;

    // term windows: every slot at the unit's first iteration, slot 0 afterwards
    if constexpr (kPacked) {
#pragma unroll
      for (int u = 0; u < kW; ++u) {
#pragma unroll
        for (int pr = 0; pr < RP; ++pr) {
          if (pr == 0 || x == xfirst) {
            const float2 rv = s_row2[pr * PS + u];
            const float cv = s_col[u];
            const float d0 = __fsub_rn(rv.x, cv), d1 = __fsub_rn(rv.y, cv);
            const float t0 = kSquare ? __fmul_rn(d0, d0) : fabsf(d0);
            const float t1 = kSquare ? __fmul_rn(d1, d1) : fabsf(d1);
            // slot 0 is refreshed; slot 1 keeps what it inherited from slot 0
            win2[pr][u] = (x == xfirst) ? f2_pack(t0, t1)
                                        : f2_pack(t0, f2_hi(win2[pr][u]));
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (r == 0 || x == xfirst) {
        if constexpr (!kDirect && kW > 0 && !kPacked) {
          if constexpr (kPair) {  // pair bits at positions TAU..kW-1 (k >= 1 only)
#pragma unroll
            for (int q = 0; q < NPH; ++q) ph[r][q] = 0u;
#pragma unroll
            for (int u = TAU; u < kW; ++u) {
              const double d0 = __dsub_rn(s_row[r * HS + u - TAU], s_col[u - TAU]);
              const double d1 = __dsub_rn(s_row[r * HS + u], s_col[u]);
              const double t0 = kSquare ? __dmul_rn(d0, d0) : fabs(d0);
              const double t1 = kSquare ? __dmul_rn(d1, d1) : fabs(d1);
              if (__dadd_rn(t0, t1) <= thr) ph[r][u >> 5] |= 1u << (u & 31);
            }
          } else if constexpr (kAnd) {
#pragma unroll
            for (int q = 0; q < NPH; ++q) ph[r][q] = 0u;
#pragma unroll
            for (int u = 0; u < kW; ++u)
              if (fabs(__dsub_rn(s_row[r * HS + u], s_col[u])) <= athr)
                ph[r][u >> 5] |= 1u << (u & 31);
          } else {
#pragma unroll
            for (int u = 0; u < kW; ++u) {
              const double d = __dsub_rn(s_row[r * HS + u], s_col[u]);
              win[r][u] = kSquare ? __dmul_rn(d, d) : fabs(d);
            }
          }
        }
      }
    }

    int kdr[R], lastc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int kd = kx - r * HS + delta;
      kdr[r] = kd;
      const int vrows = min(max(hrows - r * HS, 0), HS);
      lastc[r] = min(max(nrem - kd - r * HS, 0), vrows);  // rows of kd in slot r
    }
    // slots whose 32 diagonals all run through all HS rows: every word of the
    // iteration is a full 32-bit pass (warp-uniform fast path of the diagonal runs)
    uint32_t fullmask = 0u;
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (__all_sync(0xffffffffu, kdr[r] >= 0 && kdr[r] < nrem && lastc[r] == HS))
        fullmask |= 1u << r;

    // the R words of chunk c are final: their transposed row words go to
    // rowbuf (the R transposes are independent and interleave)
    auto chunk_rows = [&](int c, uint32_t (&w)[R]) {
      uint32_t tw[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (kdr[r] < theiler) w[r] = 0u;  // also the lower triangle kd < 0
        tw[r] = tr(w[r]);
      }
#pragma unroll
      for (int r = 0; r < R; ++r) rowbuf[wv * H + r * HS + 32 * c + lane] = tw[r];
    };
    // diagonal runs of chunks c and c+1 (64 rows per slot); one drain check
    // after every two pushes (<= 63 queued + 2 x 32 pushed < kQueueCap)
    auto diag_pass = [&](int c, const uint32_t (&w0)[R], const uint32_t (&w1)[R]) {
      if (warm || (skip & 1)) return;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int kd = kdr[r];
        if ((fullmask >> r) & 1u) {
          runs_push(w0[r], w1[r], 64, st[r], kd == 0 ? 1u : 2u, evq);
        } else {
          // past the diagonal's last row (matrix edge) nothing is consumed;
          // the piece is closed at the end of the iteration
          const bool live = kd >= 0 && kd < nrem;
          const int rel = lastc[r] - 32 * c;
          runs_push(w0[r], w1[r], live ? min(max(rel, 0), 64) : 0, st[r], kd == 0 ? 1u : 2u, evq);
        }
        if (r & 1) queue_check(evq, hist, lane);
      }
      if (R & 1) queue_check(evq, hist, lane);
    };

    if constexpr (kPre) {
      // ---- phase 1: candidate words (AND of the m shifted predicates
      // |d| <= D*) of every chunk go to this lane's rowbuf slots.  Their
      // candidates are resolved 32 at a time (exact float64 sums in the
      // reference's order) from a streaming list: per warp, nonzero words,
      // as the chunks are evaluated (m <= 4); CTA-wide, cells, after all
      // warps evaluated (m >= 5, phase 1b).  A failing candidate clears its bit.
      static_assert(R <= 4 && NCH <= 8, "candidate encoding: 2-bit slot, 3-bit chunk");
      uint16_t* cl = reinterpret_cast<uint16_t*>(smem + L.off_cand) + wv * kCandCap;
      const uint32_t wbase = smem_u32(rowbuf + wv * H);  // this warp's rowbuf words
      uint32_t lhead = 0u, ltail = 0u;  // warp-uniform list cursors
      // short sums (m <= 4): the list holds nonzero candidate WORDS (slot,
      // chunk, lane); the lane that takes an entry resolves every candidate
      // of that word and rewrites it (it is the word's only writer until
      // phase 2).  Cheaper to build than a per-cell list at the sparse
      // candidate densities where the prefilter is chosen.
      constexpr bool kWordList = (M <= 4);
      auto resolve_words = [&](uint32_t head, uint32_t avail) {
        if ((uint32_t)lane < avail) {
          const uint32_t e = cl[(head + (uint32_t)lane) & (uint32_t)(kCandCap - 1)];
          const int r = (int)(e >> 8), ce = (int)((e >> 5) & 7u), sl = (int)(e & 31u);
          const int off = r * HS + 32 * ce;
          const uint32_t addr = wbase + 4u * (uint32_t)(off + sl);
          uint32_t cand = lds_u32(addr), res = cand;
          const F* rp = s_row + off;
          const F* cp = s_col - lane + sl + 32 * ce;
          while (cand) {
            const int t = __ffs(cand) - 1;
            cand &= cand - 1u;
            if (!pre_exact(rp + t, cp + t)) res &= ~(1u << t);
          }
          asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(res) : "memory");
        }
      };
      for (int c = 0; c < NCH; ++c) {
        const F* colc = s_col + 32 * c;
        const F* rowc = s_row + 32 * c;
        if constexpr (kFP) {
          // packed float32 predicate over slot pairs; bit of step t enters
          // at bit 0 and ends at bit 31 - t (reversed after the chunk)
          const float* colf =
              reinterpret_cast<const float*>(smem + (buf ? L.off_colf1 : L.off_colf0)) +
              (int)((((uintptr_t)(a.sf + i0 + kx)) & 15u) / sizeof(float)) + delta + 32 * c;
          const unsigned long long* rowf =
              reinterpret_cast<const unsigned long long*>(smem + L.off_rowf) + 32 * c;
          const unsigned long long nd2 = f2_pack(a.pre_negd2, a.pre_negd2);
          uint32_t nw[R];
#pragma unroll
          for (int r = 0; r < R; ++r) nw[r] = 0u;
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            const float cv = colf[t + kW];
            const unsigned long long cc = f2_pack(cv, cv);
#pragma unroll
            for (int pr = 0; pr < R / 2; ++pr) {
              const unsigned long long rv = rowf[pr * (HS + W + 4) + t + kW];
              unsigned long long d, x;
              asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(rv), "l"(cc));
              asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(x) : "l"(d), "l"(nd2));
              nw[2 * pr] = __funnelshift_l((uint32_t)x, nw[2 * pr], 1);
              nw[2 * pr + 1] = __funnelshift_l((uint32_t)(x >> 32), nw[2 * pr + 1], 1);
            }
          }
          constexpr int q0 = kW >> 5, sh = kW & 31;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const uint32_t b = __brev(nw[r]);  // bit t = step t (window position t + kW)
            ph[r][q0] |= b << sh;
            if constexpr (sh != 0) ph[r][q0 + 1] |= b >> (32 - sh);
          }
        } else {
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            const double cv = colc[t + kW];
            const double cv0 = colc[t + kW - TAU];
#pragma unroll
            for (int r = 0; r < R; ++r) {
              // pair (position t + kW - TAU, t + kW), in the reference's term form
              const double d0 = __dsub_rn(rowc[r * HS + t + kW - TAU], cv0);
              const double d1 = __dsub_rn(rowc[r * HS + t + kW], cv);
              const double t0 = kSquare ? __dmul_rn(d0, d0) : fabs(d0);
              const double t1 = kSquare ? __dmul_rn(d1, d1) : fabs(d1);
              if (__dadd_rn(t0, t1) <= thr) ph[r][(t + kW) >> 5] |= 1u << ((t + kW) & 31);
            }
          }
        }
        uint32_t wr[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          // component predicates: AND over k = 0..m-1; pair predicates: the
          // m-1 pairs (k-1, k) sit at positions k * TAU, k = 1..m-1
          uint32_t w = kPair ? 0xffffffffu : ph[r][0];
#pragma unroll
          for (int k = 1; k < M; ++k)
            w &= __funnelshift_rc(ph[r][(k * TAU) >> 5], ph[r][((k * TAU) >> 5) + 1],
                                  (k * TAU) & 31);
#pragma unroll
          for (int q = 0; q + 1 < NPH; ++q) ph[r][q] = ph[r][q + 1];
          ph[r][NPH - 1] = 0u;
          w = kdr[r] < theiler ? 0u : w;  // Theiler-excluded cells need no sum
          wr[r] = w;
          asm volatile("st.shared.u32 [%0], %1;" ::"r"(rowbuf_sa + 4u * (uint32_t)(r * HS + 32 * c)),
                       "r"(w)
                       : "memory");
        }
        if constexpr (kWordList) {
          // at most R * 32 new entries per chunk: the list never overflows;
          // the previous round's reads of reused ring entries come first
          __syncwarp();
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const uint32_t mk = __ballot_sync(0xffffffffu, wr[r] != 0u);
            if (wr[r] != 0u)
              cl[(ltail + __popc(mk & evq.lt_mask)) & (uint32_t)(kCandCap - 1)] =
                  (uint16_t)((r << 8) | (c << 5) | lane);
            ltail += __popc(mk);
          }
          RQA_DCHECK(ltail - lhead <= (uint32_t)kCandCap);
          __syncwarp();
          while (ltail - lhead >= 32u) {
            resolve_words(lhead, 32u);
            lhead += 32u;
          }
          continue;
        }
      }
      if constexpr (kWordList) {
        __syncwarp();
        while (ltail != lhead) {  // the last, partial round
          const uint32_t avail = min(ltail - lhead, 32u);
          resolve_words(lhead, avail);
          lhead += avail;
        }
        __syncwarp();
      } else {
        // ---- phase 1b (long sums): the candidate cells of the whole CTA are
        // resolved by all warps.  Word group g = (source warp ws, slot r,
        // chunk c) goes to warp (ws + r * NCH + c) % NW, so every warp gets an
        // equal share of every source warp's groups (the candidate density
        // varies across diagonals, i.e. across warps).  Entries: group index
        // gi = r * NCH + c (5 bits), lane, step.
        static_assert(R * NCH <= 32 && (NW & (NW - 1)) == 0, "group encoding");
        __syncthreads();  // every warp's candidate words are in rowbuf
        const F* colbase = s_col - delta;  // column window of lane 0 of warp 0
        auto resolve_cells = [&](uint32_t head, uint32_t avail) {
          if ((uint32_t)lane < avail) {
            const uint32_t e = cl[(head + (uint32_t)lane) & (uint32_t)(kCandCap - 1)];
            const int gi = (int)(e >> 10), sl = (int)((e >> 5) & 31u), t = (int)(e & 31u);
            const int r = gi / NCH, ce = gi % NCH, ws = (wv - gi) & (NW - 1);
            const int off = r * HS + 32 * ce;
            if (!pre_exact(s_row + off + t, colbase + 32 * ws + sl + 32 * ce + t)) {
              const uint32_t addr = smem_u32(rowbuf + ws * H + off + sl);
              asm volatile("red.shared.and.b32 [%0], %1;" ::"r"(addr), "r"(~(1u << t)) : "memory");
            }
          }
        };
#pragma unroll 1
        for (int gi = 0; gi < R * NCH; ++gi) {
          const int r = gi / NCH, ce = gi % NCH, ws = (wv - gi) & (NW - 1);
          const int off = r * HS + 32 * ce;
          // the last round's list reads precede this group's appends, which
          // may reuse those ring entries (compute-sanitizer racecheck)
          __syncwarp();
          const uint32_t w = rowbuf[ws * H + off + lane];
          const int kr = __popc(w);
          int incl = kr;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
          }
          const uint32_t tot = (uint32_t)__shfl_sync(0xffffffffu, incl, 31);
          if (ltail - lhead + tot <= (uint32_t)kCandCap) {
            uint32_t pos = ltail + (uint32_t)(incl - kr);
            uint32_t ww = w;
            while (ww) {
              const int t = __ffs(ww) - 1;
              ww &= ww - 1u;
              cl[pos++ & (uint32_t)(kCandCap - 1)] = (uint16_t)((gi << 10) | (lane << 5) | t);
            }
            ltail += tot;
            RQA_DCHECK(ltail - lhead <= (uint32_t)kCandCap);
            __syncwarp();
            while (ltail - lhead >= 32u) {
              resolve_cells(lhead, 32u);
              lhead += 32u;
            }
          } else {
            // dense word set: every lane resolves its own word of the group
            uint32_t cand = w, res = w;
            while (cand) {
              const int t = __ffs(cand) - 1;
              cand &= cand - 1u;
              if (!pre_exact(s_row + off + t, colbase + 32 * ws + lane + 32 * ce + t))
                res &= ~(1u << t);
            }
            rowbuf[ws * H + off + lane] = res;
          }
        }
        __syncwarp();
        while (ltail != lhead) {  // the last, partial round
          const uint32_t avail = min(ltail - lhead, 32u);
          resolve_cells(lhead, avail);
          lhead += avail;
        }
        __syncthreads();  // resolved words visible to their owners
      }
      // ---- phase 2: final words -> transposed row words, diagonal runs
      static_assert(NCH % 2 == 0, "chunk pairs");
      for (int c = 0; c < NCH; c += 2) {
        uint32_t w0[R], w1[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          w0[r] = lds_u32(rowbuf_sa + 4u * (uint32_t)(r * HS + 32 * c));
          w1[r] = lds_u32(rowbuf_sa + 4u * (uint32_t)(r * HS + 32 * c + 32));
        }
        chunk_rows(c, w0);
        chunk_rows(c + 1, w1);
        diag_pass(c, w0, w1);
      }
    } else {
    uint32_t wprev[R];  // words of the even chunk of a pair (diagonal runs per chunk pair)
    for (int c = 0; c < NCH; ++c) {
      uint32_t dw[R];
      float amb[R];  // f32 filter: min |acc32 - c32| over the word (per pair when packed)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        dw[r] = 0u;
        amb[r] = __int_as_float(0x7f800000);
      }
      const F* colc = s_col + 32 * c;
      const F* rowc = s_row + 32 * c;
      if constexpr (kPacked) {
        const unsigned long long negc = f2_pack(-a.c32, -a.c32);
#pragma unroll
        for (int t = 0; t < 32; ++t) {
          const float cv = colc[t + kW];
          const unsigned long long negcv = f2_pack(-cv, -cv);
#pragma unroll
          for (int pr = 0; pr < RP; ++pr) {
            const float2 rv = s_row2[pr * PS + 32 * c + t + kW];
            const unsigned long long d = f2_add(f2_pack(rv.x, rv.y), negcv);
            const unsigned long long term = kSquare ? f2_mul(d, d) : (d & 0x7fffffff7fffffffull);
            unsigned long long acc = win2[pr][0];
#pragma unroll
            for (int k = 1; k < M - 1; ++k) acc = f2_add(acc, win2[pr][k * TAU]);
            acc = f2_add(acc, term);
            const unsigned long long xx = f2_add(acc, negc);
            // sign of acc32 - c32 (exact) shifted in; bit t ends at 31 - t
            dw[2 * pr] = __funnelshift_l(__float_as_uint(f2_lo(xx)), dw[2 * pr], 1);
            dw[2 * pr + 1] = __funnelshift_l(__float_as_uint(f2_hi(xx)), dw[2 * pr + 1], 1);
            amb[pr] = fminf(amb[pr], fminf(fabsf(f2_lo(xx)), fabsf(f2_hi(xx))));
#pragma unroll
            for (int j = 0; j + 1 < kW; ++j) win2[pr][j] = win2[pr][j + 1];
            win2[pr][kW - 1] = term;
          }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) dw[r] = __brev(dw[r]);
      } else
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        if constexpr (kF32) {  // direct f32 evaluation (runtime m, tau)
          const int m = a.m, tau = a.tau;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const float* rp = reinterpret_cast<const float*>(rowc) + r * HS + t;
            const float* cp = reinterpret_cast<const float*>(colc) + t;
            bool hit;
            if (METRIC == kLinf || m == 1) {
              hit = true;
              for (int k = 0; k < m; ++k) {
                const float ad = fabsf(__fsub_rn(rp[k * tau], cp[k * tau]));
                hit &= ad <= a.thr32;
                amb[r] = fminf(amb[r], fabsf(__fsub_rn(ad, a.c32)));
              }
            } else {
              float acc = 0.0f;
              for (int k = 0; k < m; ++k) {
                const float d = __fsub_rn(rp[k * tau], cp[k * tau]);
                const float term = (METRIC == kL2) ? __fmul_rn(d, d) : fabsf(d);
                acc = (k == 0) ? term : __fadd_rn(acc, term);
              }
              hit = acc <= a.thr32;
              amb[r] = fminf(amb[r], fabsf(__fsub_rn(acc, a.c32)));
            }
            if (hit) dw[r] |= 1u << t;
          }
        } else if constexpr (!kDirect) {
          const double cv = colc[t + kW];
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const double rv = rowc[r * HS + t + kW];
            const double d = __dsub_rn(rv, cv);
            if constexpr (M == 1) {
              setbit_le(dw[r], fabs(d), thr, 1u << t);
            } else if constexpr (kAnd) {
              if (fabs(d) <= athr) {
                ph[r][(t + kW) >> 5] |= 1u << ((t + kW) & 31);
              }
            } else {
              const double term = kSquare ? __dmul_rn(d, d) : fabs(d);
              double acc = win[r][0];
#pragma unroll
              for (int k = 1; k < M - 1; ++k) acc = __dadd_rn(acc, win[r][k * TAU]);
              acc = __dadd_rn(acc, term);
              setbit_le(dw[r], acc, thr, 1u << t);
#pragma unroll
              for (int j = 0; j + 1 < kW; ++j) win[r][j] = win[r][j + 1];
              win[r][kW - 1] = term;
            }
          }
        } else {
          const int m = a.m, tau = a.tau;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const double* rp = rowc + r * HS + t;
            const double* cp = colc + t;
            bool hit;
            if (METRIC == kLinf || m == 1) {
              hit = true;
              for (int k = 0; k < m; ++k) hit &= (fabs(__dsub_rn(rp[k * tau], cp[k * tau])) <= thr);
            } else {
              double acc = 0.0;
              for (int k = 0; k < m; ++k) {
                const double d = __dsub_rn(rp[k * tau], cp[k * tau]);
                const double term = (METRIC == kL2) ? __dmul_rn(d, d) : fabs(d);
                acc = (k == 0) ? term : __dadd_rn(acc, term);
              }
              hit = acc <= thr;
            }
            if (hit) dw[r] |= 1u << t;
          }
        }
      }

      if constexpr (kF32) {
        // words with a cell inside the band: float64 bits (exact mode) or the
        // float32 bits plus the fp32/fp64 mismatch count (fp32 mode)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const float am = kPacked ? amb[r / 2] : amb[r];
          if (a.all_amb || am <= a.band32) {
            const int kd = kdr[r];
            const uint2 w = f32_recheck<METRIC>(a, i0 + r * HS + 32 * c, (int64_t)kd);
            if (a.prec_mode == 0) {
              dw[r] = w.x;
            } else {
              dw[r] = w.y;
              if (!warm && kd >= theiler && kd < nrem) {
                const uint32_t mk = low_mask(min(max(lastc[r] - 32 * c, 0), 32));
                mism += (unsigned long long)((kd == 0) ? 1 : 2) * __popc((w.x ^ w.y) & mk);
              }
            }
          }
        }
      }
      uint32_t words[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if constexpr (kAnd) {  // L-inf: AND of the m shifted per-component predicates
          uint32_t word = ph[r][0];
#pragma unroll
          for (int k = 1; k < M; ++k)
            word &= __funnelshift_rc(ph[r][(k * TAU) >> 5], ph[r][((k * TAU) >> 5) + 1],
                                     (k * TAU) & 31);
#pragma unroll
          for (int q = 0; q + 1 < NPH; ++q) ph[r][q] = ph[r][q + 1];
          ph[r][NPH - 1] = 0u;
          words[r] = word;
        } else {
          words[r] = dw[r];
        }
      }
      chunk_rows(c, words);
      if (c & 1) {
        diag_pass(c - 1, wprev, words);
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) wprev[r] = words[r];
      }
    }
    }
    __syncthreads();

    // ---- row phase (not in the recomputed iteration): row parts of hooks
    const uint32_t* prev_cur = prevbuf + buf * H;    // words of iteration x-1, warp NW-1
    uint32_t* prev_next = prevbuf + (buf ^ 1) * H;
    constexpr int PR = (R % 2 == 0) ? 2 : 1;  // slot pairs (column phase)
    // rows per thread handled together in the row phase (independent run
    // states interleave; a drain check after every two passes): all R slots
    // for the prefilter kernels (sparse by construction: C3 -0.45 %), pairs
    // otherwise (dense data, P: 4 measured +2 %)
    constexpr int PRR = (PREC == 2 && R % 4 == 0) ? 4 : PR;
#pragma unroll 1
    for (int r0 = 0; r0 < R; r0 += PRR) {
      int lr[PRR], rem[PRR];
      RunState rs[PRR];
      bool any_rem = false, all_full = true;
#pragma unroll
      for (int p = 0; p < PRR; ++p) {
        const int r = r0 + p;
        lr[p] = r * HS + tid;
        prev_next[lr[p]] = rowbuf[(NW - 1) * H + lr[p]];
        const bool act = !warm && x >= r && lr[p] < hrows;
        rem[p] = act ? nrem - lr[p] - (x - r) * D : 0;
        any_rem |= rem[p] > 0;
        all_full &= rem[p] >= D;
      }
      if (!(skip & 2) && __any_sync(0xffffffffu, any_rem)) {
#pragma unroll
        for (int p = 0; p < PRR; ++p) {
          const uint2 rsv = rowst[lr[p]];
          rs[p] = RunState{rsv.x, rsv.y};
        }
        if (__all_sync(0xffffffffu, all_full)) {
          static_assert(NW % 2 == 0, "row phase: word pairs");
#pragma unroll 1
          for (int v = 0; v < NW; v += 2) {
#pragma unroll
            for (int p = 0; p < PRR; ++p) {
              const uint32_t w0 = rowbuf[v * H + lr[p]], w1 = rowbuf[(v + 1) * H + lr[p]];
              pts += __popc(w0) + __popc(w1);
              runs_push(w0, w1, 64, rs[p], 0u, evq);
              if (p % 2 == 1 || p == PRR - 1) queue_check(evq, hist, lane);
            }
          }
        } else {
#pragma unroll 1
          for (int v = 0; v < NW; v += 2) {
#pragma unroll
            for (int p = 0; p < PRR; ++p) {
              const int nb = min(max(rem[p] - 32 * v, 0), 64);
              const uint32_t w0 = rowbuf[v * H + lr[p]] & low_mask(nb);
              const uint32_t w1 = rowbuf[(v + 1) * H + lr[p]] & (nb > 32 ? low_mask(nb - 32) : 0u);
              pts += __popc(w0) + __popc(w1);
              runs_push(w0, w1, nb, rs[p], 0u, evq);
              if (p % 2 == 1 || p == PRR - 1) queue_check(evq, hist, lane);
            }
          }
        }
#pragma unroll
        for (int p = 0; p < PRR; ++p) {
          const int r = r0 + p;
          if (rem[p] > 0 && x == r) pts64 -= (rowbuf[lr[p]] & 1u);  // diagonal cell once
          rowst[lr[p]] = make_uint2(rs[p].first, rs[p].cur);
        }
      }
    }
    pts64 += 2ull * pts;
    pts = 0;

    // ---- column phase: finishing blocks (not in the recomputed iteration) and
    // starting blocks (not in the last iteration: the next unit owns them)
    {
      const bool do_fin = !warm;
      const bool do_new = x + 1 < xb;
      Seg acc{0u, 0u, 0u};
      const int cfin = kx + 32 * wv + lane;
      const int cnew = cfin + D;
#ifndef RQA_COL_PR
#define RQA_COL_PR 2
#endif
      // slots handled together in the column phase
      constexpr int PC = (R % RQA_COL_PR == 0) ? RQA_COL_PR : PR;
#pragma unroll 1
      for (int rr0 = 0; rr0 < R; rr0 += PC) {
        int rs_[PC], lim_fin[PC], lim_new[PC];
        RunState cur[PC], nst[PC], fin[PC];
#pragma unroll
        for (int p = 0; p < PC; ++p) {
          const int r = R - 1 - (rr0 + p);
          rs_[p] = r;
          const uint2 cs = colst[(wv * R + r) * 32 + lane];
          fin[p] = RunState{cs.y, cs.x};
          nst[p] = RunState{0u, 0u};
          cur[p] = RunState{0u, 0u};
          lim_fin[p] = (do_fin && x >= r && cfin < nrem) ? min(cfin, hrows) - r * HS : 0;
          lim_new[p] = (do_new && x >= r && cnew < nrem) ? min(cnew, hrows) - r * HS : 0;
        }
        if (!(skip & 4) && x >= rs_[PC - 1]) {
          // column window c of slot rows: words of warps wp-1 and wp funnel-
          // shifted into aligned columns, transposed, bit-reversed (columns
          // are met bottom-up); all lanes take part (transpose)
          auto col_word = [&](int c, int p) {
            const int wp = (wv - c) & (NW - 1);
            const int lrow = rs_[p] * HS + 32 * c + lane;
            const uint32_t w1 = rowbuf[wp * H + lrow];
            const uint32_t w0 = wp > 0 ? rowbuf[(wp - 1) * H + lrow] : prev_cur[lrow];
            return __brev(tr(__funnelshift_l(w0, w1, lane)));
          };
          // windows c and c-1 (c-1 < lo: none) as one 64-bit pass per slot;
          // partial columns keep the rows below lim (a window's valid rows are
          // its top ones: after the bit reversal, its high bits)
          auto col_pair = [&](int c, int lo, const int* lim, auto full) {
#pragma unroll
            for (int p = 0; p < PC; ++p) {
              const uint32_t a0 = col_word(c, p);
              const uint32_t a1 = c - 1 >= lo ? col_word(c - 1, p) : 0u;
              if constexpr (decltype(full)::value) {  // every lane: 32 rows per window
                runs_push(a0, a1, c - 1 >= lo ? 64 : 32, cur[p], 0u, evq);
              } else {
                const int n0 = min(max(lim[p] - 32 * c, 0), 32);
                const int n1 = c - 1 >= lo ? min(max(lim[p] - 32 * (c - 1), 0), 32) : 0;
                const uint32_t b0 = __funnelshift_rc(a0, 0u, 32 - n0);
                const uint32_t b1 = __funnelshift_rc(a1, 0u, 32 - n1);
                const unsigned long long x64 = (unsigned long long)b0 |
                                               ((unsigned long long)b1 << n0);
                runs_push((uint32_t)x64, (uint32_t)(x64 >> 32), n0 + n1, cur[p], 0u, evq);
              }
              if (p % 2 == 1 || p == PC - 1) queue_check(evq, hist, lane);
            }
          };
          // windows c = hi, hi-1, ..., lo (descending), two per pass
          auto col_steps = [&](int hi, int lo, const int* lim, auto full) {
#pragma unroll 1
            for (int c = hi; c >= lo; c -= 2) col_pair(c, lo, lim, full);
          };
          using kFull = std::integral_constant<bool, true>;
          using kPart = std::integral_constant<bool, false>;
          bool fnew = true, ffin = true;
#pragma unroll
          for (int p = 0; p < PC; ++p) {
            fnew &= lim_new[p] >= 32 * NCH;
            ffin &= lim_fin[p] >= 32 * (wv + 1);
          }
          fnew = __all_sync(0xffffffffu, fnew);
          ffin = __all_sync(0xffffffffu, ffin);
          // windows above the warp's own start the columns of iteration x+1
          if (do_new) {
            if (fnew) col_steps(NCH - 1, wv + 1, lim_new, kFull{});
            else col_steps(NCH - 1, wv + 1, lim_new, kPart{});
          }
#pragma unroll
          for (int p = 0; p < PC; ++p) {
            nst[p] = cur[p];
            cur[p] = fin[p];
          }
          // the warp's own window and those below finish the columns of x
          if (do_fin) {
            if (ffin) col_steps(wv, 0, lim_fin, kFull{});
            else col_steps(wv, 0, lim_fin, kPart{});
          }
#pragma unroll
          for (int p = 0; p < PC; ++p) fin[p] = cur[p];
        }
#pragma unroll
        for (int p = 0; p < PC; ++p) {
          acc = seg_combine(acc, runs_finish(fin[p]), hist);
          colst[(wv * R + rs_[p]) * 32 + lane] = make_uint2(nst[p].cur, nst[p].first);
        }
      }
      if (do_fin && cfin < nrem) RQA_DCHECK(cfin >= 0 && (Cb - a.colsum) + cfin < ua.cap_cs);
      if (do_fin && cfin < nrem)
        Cb[cfin] = (cfin == 0) ? 0u
                 : acc.uniform ? pack_col(acc.first, acc.first)
                               : pack_col(acc.last, acc.first);
    }
    __syncthreads();

    // ---- diagonal pieces: a band segment ends in the slot holding its last
    // row (open: the band's last row, it may continue in the next band;
    // closed: cut by the matrix's right edge); a segment that continues past
    // the unit's last iteration is handed to the next unit through drec
    if (!warm) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int kd = kdr[r];
        if (kd >= 0 && kd < nrem) {
          const int brows = min(hrows, nrem - kd);  // rows of kd in this band
          // slot r ends the segment iff its last row lies in slot r.  The
          // prefilter and L-inf kernels test the range of brows - 1 - r * HS:
          // with r == (brows-1)/HS ptxas indexes st[] by the quotient and
          // moves it to local memory (range test: C3 -1.75 %, C5 -0.27 %,
          // C4 -0.3 %); the float64 term-reuse kernels keep the quotient (P
          // measured +0.9 % with the range test)
          const int lrow = brows - 1 - r * HS;
          const int rend = (brows - 1) / HS;
          if (kRangeEnd ? (lrow >= 0 && lrow < HS) : r == rend) {
            const uint32_t ps = diag_piece_end(st[r], brows == hrows,
                                               LineSink{&hist, kd == 0 ? 1u : 2u});
            if (x - r >= xa) {  // the whole band segment was walked by this unit
              RQA_DCHECK((Pb - a.P) + kd < ua.cap_ps);
              Pb[kd] = (uint16_t)(ps & 0xffffu);
              Sb[kd] = (uint16_t)(ps >> 16);
            } else {  // lower part of a segment cut at xa (upper part: unit idx-1)
              RQA_DCHECK(unit.idx >= 1 && xa - 1 - (x - r) >= 0 && xa - 1 - (x - r) < R - 1 &&
                         ((int64_t)(unit.idx - 1) * (R - 1) + (xa - 1 - (x - r))) * D + delta <
                             ua.cap_drec);
              ua.drec[((int64_t)(unit.idx - 1) * (R - 1) + (xa - 1 - (x - r))) * D + delta].y =
                  ps | (brows == hrows ? 0u : 0x80000000u);
            }
          } else if ((kRangeEnd ? lrow >= HS : r < rend) && x == xb - 1) {  // upper part of a segment cut at xb
            RQA_DCHECK(r < R - 1 && ((int64_t)unit.idx * (R - 1) + r) * D + delta < ua.cap_drec);
            ua.drec[((int64_t)unit.idx * (R - 1) + r) * D + delta].x =
                diag_piece_end(st[r], true, LineSink{&hist, 0u});
          }
        }
      }
    }
    // slot r+1 walks slot r's diagonals in the next iteration
#pragma unroll
    for (int r = R - 1; r >= 1; --r) st[r] = st[r - 1];
    st[0] = RunState{0u, 0u};
    if constexpr (kPacked) {  // slot r+1 continues slot r's window (pairs: lo = even slot)
#pragma unroll
      for (int j = 0; j < kW; ++j) {
#pragma unroll
        for (int pr = RP - 1; pr >= 0; --pr) {
          const uint32_t lo_new = pr > 0 ? (uint32_t)(win2[pr - 1][j] >> 32) : 0u;
          win2[pr][j] = ((unsigned long long)(uint32_t)win2[pr][j] << 32) | lo_new;
        }
      }
    }
#pragma unroll
    for (int r = R - 1; r >= 1; --r) {
      if constexpr (!kDirect && kW > 0 && !kPacked) {
        if constexpr (kAnd) {
#pragma unroll
          for (int q = 0; q < NPH; ++q) ph[r][q] = ph[r - 1][q];
        } else {
#pragma unroll
          for (int j = 0; j < kW; ++j) win[r][j] = win[r - 1][j];
        }
      }
    }
    if (((it + 1) & a.flush_mask) == 0) {
      // 32-bit shared bins are emptied into the 64-bit histogram every 4096
      // iterations (no overflow); first every warp's adds of this iteration
      // (the diagonal pieces closed above) must have landed
      __syncthreads();
      for (int q = tid; q < 3 * kSmemBins; q += NW * 32) {
        const uint32_t cnt = sh_hist[q];
        if (cnt) {
          atomicAdd(&a.hist[(q / kSmemBins) * (n + 1) + (q % kSmemBins)], (unsigned long long)cnt);
          sh_hist[q] = 0u;
        }
      }
      __syncthreads();
    }
  }

  // ---- row pieces of this unit: (first, last) runs, read by the hook fold
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int lr = r * HS + tid;
    if (lr < hrows) {
      const uint2 rsv = rowst[lr];
      const Seg sg = runs_finish(RunState{rsv.x, rsv.y});
      RQA_DCHECK((int64_t)unit.idx * H + lr < ua.cap_piece);
      piece[lr] = make_uint2(sg.first, sg.last);
    }
  }

  queue_drain(evq, hist, lane, true);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) pts64 += __shfl_xor_sync(0xffffffffu, pts64, o);
  if (lane == 0 && pts64) atomicAdd(a.points, pts64);
  if constexpr (kF32) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) mism += __shfl_xor_sync(0xffffffffu, mism, o);
    if (lane == 0 && mism) atomicAdd(a.mism, mism);
  }
  __syncthreads();
  for (int q = tid; q < 3 * kSmemBins; q += NW * 32) {
    const uint32_t cnt = sh_hist[q];
    if (cnt) atomicAdd(&a.hist[(q / kSmemBins) * (n + 1) + (q % kSmemBins)], (unsigned long long)cnt);
  }
}

}  // namespace rqa
