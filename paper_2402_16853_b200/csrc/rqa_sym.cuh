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

struct SymSmem {
  int H, HS, D, W, CW;
  size_t off_row, off_col0, off_col1, off_rowbuf, off_prev, off_colst, off_rowst, off_queue,
      off_hist, total;
  // esize 8: float64 row/column windows; 4: float32 windows (f32 filter
  // kernels), the row window stored as R/2 interleaved slot pairs of
  // HS + W + 4 float2 each (rqa_unit.cuh, packed f32x2 evaluation).
  __host__ __device__ SymSmem(int NW, int R, int W_, int esize = 8) {
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
    off_queue = off_rowst + (size_t)R * D * sizeof(uint2);
    off_hist = off_queue + (size_t)NW * kQueueCap * sizeof(uint4);
    total = off_hist + 3 * kSmemBins * sizeof(uint32_t) + 16;
  }
};

// Set bit T of dw iff acc <= thr: DSETP + predicated LOP3 (no SEL chains).
__device__ __forceinline__ void setbit_le(uint32_t& dw, double acc, double thr, uint32_t bit) {
  asm("{\n\t.reg .pred p;\n\tsetp.le.f64 p, %1, %2;\n\t@p or.b32 %0, %0, %3;\n\t}"
      : "+r"(dw)
      : "d"(acc), "d"(thr), "r"(bit));
}

// A diagonal's segment inside the band ends: report its band-top run as P
// (length if it is a run of ones, else 0) and, if the segment ends at the
// band's bottom edge (open), its bottom run as S; a segment cut by the
// matrix's right edge (closed) counts its last run here.
__device__ __forceinline__ void diag_finish(const RunState& st, bool open, uint16_t* Pk,
                                            uint16_t* Sk, const LineSink& sink) {
  const Seg g = runs_finish(st);
  const uint32_t first = g.first;
  *Pk = (uint16_t)(run_bit(first) ? run_len(first) : 0u);
  if (open) {
    *Sk = (uint16_t)(run_bit(g.last) ? run_len(g.last) : 0u);
  } else if (!g.uniform) {
    sink(g.last);
  }
}

template <int METRIC, int M, int TAU, int NW, int R, int MINB>
__global__ void __launch_bounds__(NW * 32, MINB)
sym_kernel(const SymArgs a, const int W_rt) {
  constexpr int D = 32 * NW;
  constexpr int HS = D;
  constexpr int H = R * HS;
  constexpr bool kDirect = (M == 0);
  constexpr int kW = kDirect ? 0 : (M - 1) * TAU;
  constexpr bool kLinfAnd = (METRIC == kLinf) && (M >= 2);
  constexpr bool kSquare = (METRIC == kL2) && (M >= 2);
  constexpr int NCH = HS / 32;  // == NW
  static_assert(kLinfAnd ? kW <= 32 : kW <= 48, "term window too large");
  const int W = kDirect ? W_rt : kW;
  const SymSmem L(NW, R, W);

  extern __shared__ __align__(128) unsigned char smem[];
  double* s_row = reinterpret_cast<double*>(smem + L.off_row);
  uint32_t* rowbuf = reinterpret_cast<uint32_t*>(smem + L.off_rowbuf);
  uint32_t* prevbuf = reinterpret_cast<uint32_t*>(smem + L.off_prev);
  uint2* colst = reinterpret_cast<uint2*>(smem + L.off_colst);
  uint2* rowst = reinterpret_cast<uint2*>(smem + L.off_rowst);  // row-part run state (first, cur)
  uint32_t* sh_hist = reinterpret_cast<uint32_t*>(smem + L.off_hist);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L.off_hist + 3 * kSmemBins * sizeof(uint32_t));

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int wv = tid >> 5;
  const int delta = 32 * wv + lane;
  const int64_t n = a.n;
  const int64_t b = blockIdx.x;
  const int64_t i0 = a.row_lo + b * H;
  const int64_t i_end = min(i0 + (int64_t)H, a.row_hi);
  const int nrem = (int)(n - i0);                  // diagonals (and columns) present in the band
  const int X = (nrem + D - 1) / D + R - 1;
  const int hrows = (int)(i_end - i0);             // valid rows of the band
  const int bot_rows = (int)(n - i_end) + 1;       // kd < bot_rows <=> bottom row valid
  const int theiler = (int)min(a.theiler, (int64_t)1 << 30);
  const double thr = a.thr;
  const int64_t boff = band_offset(b, n, a.row_lo, H);
  uint16_t* Pb = a.P + boff;
  uint16_t* Sb = a.S + boff;
  uint32_t* Cb = a.colsum + boff;
  uint32_t* lead_out = a.rowlead + i0;
  const Hist hist{smem_u32(sh_hist), a.hist, n + 1};
  const Transposer tr(lane);
  EventQueue evq{reinterpret_cast<uint4*>(smem + L.off_queue) + wv * kQueueCap, 0u, 0u,
                 (1u << lane) - 1u};
  evq.ring_sa = smem_u32(evq.ring);

  for (int q = tid; q < 3 * kSmemBins; q += NW * 32) sh_hist[q] = 0u;
  for (int q = tid; q < H + W; q += NW * 32) s_row[q] = a.s[i0 + q];
  for (int q = tid; q < 2 * H; q += NW * 32) prevbuf[q] = 0u;
  for (int q = tid; q < NW * R * 32; q += NW * 32) colst[q] = make_uint2(0u, 0u);
  for (int q = tid; q < R * D; q += NW * 32) rowst[q] = make_uint2(0u, 0u);
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t col_bytes = (uint32_t)(L.CW * sizeof(double));
  if (tid == 0) {
    const double* src;
    col_window_src(a.s, i0, &src);
    mbar_expect_tx_arrive(&bar[0], col_bytes);
    tma_load_1d(smem + L.off_col0, src, col_bytes, &bar[0]);
  }

  // profiling experiment: offset CTAs so co-resident CTAs are out of phase
  if (a.skip & 8) { if ((blockIdx.x & 1) && tid == 0) __nanosleep(13000); __syncthreads(); }
  if (a.skip & 16) { if (((blockIdx.x / 148) & 1) && tid == 0) __nanosleep(13000); __syncthreads(); }
  RunState st[R];  // diagonal run state per slot (first run = band-top run)
  double win[R][kW > 0 ? kW : 1];
  uint32_t ph_lo[R], ph_hi[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    st[r] = RunState{0u, 0u};
    ph_lo[r] = 0u;
    ph_hi[r] = 0u;
  }
  const LineSink vsink{&hist, 0u};
  uint32_t pts = 0;  // per-thread partial, flushed to 64 bits every iteration

  unsigned long long pts64 = 0;
  unsigned long long tm[4] = {0, 0, 0, 0};
  long long tprev = clock64();
  for (int x = 0; x < X; ++x) {
    const int kx = x * D;
    const int buf = x & 1;
    if (tid == 0 && x + 1 < X) {
      const double* src;
      col_window_src(a.s, i0 + kx + D, &src);
      mbar_expect_tx_arrive(&bar[buf ^ 1], col_bytes);
      tma_load_1d(smem + (buf ? L.off_col0 : L.off_col1), src, col_bytes, &bar[buf ^ 1]);
    }
    mbar_wait(&bar[buf], (uint32_t)((x >> 1) & 1));
    const int co = (int)((((uintptr_t)(a.s + i0 + kx)) >> 3) & 1);
    const double* s_col =
        reinterpret_cast<const double*>(smem + (buf ? L.off_col1 : L.off_col0)) + co + delta;

    // ---- warm-up of fresh slots ------------------------------------------
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (r == 0 || x == 0) {
        st[r] = RunState{0u, 0u};
        if constexpr (!kDirect && kW > 0) {
          if constexpr (kLinfAnd) {
            uint32_t p = 0;
#pragma unroll
            for (int u = 0; u < kW; ++u)
              if (fabs(__dsub_rn(s_row[r * HS + u], s_col[u])) <= thr) p |= 1u << u;
            ph_lo[r] = p;
            ph_hi[r] = 0u;
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

    // per-slot geometry of this iteration, relative to the slot's first row
    int kdr[R];     // kd of this lane's diagonal in slot r (may be < 0)
    int lastc[R];   // rows [0, lastc) of slot r are valid cells of the diagonal
    int openb[R];   // 1: the diagonal continues past the slot's valid rows into the next band
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int kd = kx - r * HS + delta;
      kdr[r] = kd;
      const int vrows = min(max(hrows - r * HS, 0), HS);
      const int crows = min(max(nrem - kd - r * HS, 0), vrows);
      lastc[r] = crows;
      openb[r] = (crows == vrows) ? 1 : 0;
    }

    // Bookkeeping of one finished chunk cc (its R words): diagonal runs,
    // row words to shared memory.  Software-pipelined: chunk c-1 is booked
    // inside the same basic block as chunk c's FP64 steps so the scheduler
    // can overlap the integer work with the FP64 pipe.
    auto book = [&](int cc, const uint32_t (&words)[R], bool valid) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int kd = kdr[r];
        const bool live = valid && kd >= 0 && kd < nrem;
        const int rel = lastc[r] - 32 * cc;
        if (!(a.skip & 1))
          runs_pass(words[r], live ? min(max(rel, 0), 32) : 0, st[r], kd == 0 ? 1u : 2u, evq,
                    hist, lane);
        const uint32_t rw = tr(words[r]);
        if (valid) rowbuf[wv * H + r * HS + 32 * cc + lane] = rw;
      }
    };
    // the segment of slot r is cut by the matrix's right edge in this chunk
    auto close_cut = [&](int cc) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int kd = kdr[r];
        const int rel = lastc[r] - 32 * cc;
        if (kd >= 0 && kd < nrem && !openb[r] && rel >= 0 && rel < 32 && st[r].cur != 0u) {
          diag_finish(st[r], false, Pb + kd, Sb + kd, LineSink{&hist, kd == 0 ? 1u : 2u});
          st[r] = RunState{1u, 0u};  // finished: later slots of this diagonal are empty
        }
      }
    };

    uint32_t pw[R];
#pragma unroll
    for (int r = 0; r < R; ++r) pw[r] = 0u;
    for (int c = 0; c < NCH; ++c) {
      uint32_t dw[R];
#pragma unroll
      for (int r = 0; r < R; ++r) dw[r] = 0u;
      const double* colc = s_col + 32 * c;
      const double* rowc = s_row + 32 * c;
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        if constexpr (!kDirect) {
          const double cv = colc[t + kW];
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const double rv = rowc[r * HS + t + kW];
            const double d = __dsub_rn(rv, cv);
            if constexpr (M == 1) {
              setbit_le(dw[r], fabs(d), thr, 1u << t);
            } else if constexpr (kLinfAnd) {
              if (fabs(d) <= thr) {
                if (t + kW < 32) ph_lo[r] |= 1u << ((t + kW) & 31);
                else ph_hi[r] |= 1u << ((t + kW - 32) & 31);
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
      // finalise this chunk's words (Linf AND of shifted predicates, Theiler band)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        uint32_t word;
        if constexpr (kLinfAnd) {
          word = ph_lo[r];
#pragma unroll
          for (int k = 1; k < M; ++k) word &= __funnelshift_rc(ph_lo[r], ph_hi[r], k * TAU);
          ph_lo[r] = ph_hi[r];
          ph_hi[r] = 0u;
        } else {
          word = dw[r];
        }
        pw[r] = (kdr[r] < theiler) ? 0u : word;  // also the lower triangle kd < 0
      }
      book(c, pw, true);
      close_cut(c);
      if (evq.tail - evq.head >= 32u) queue_drain(evq, hist, lane, false);
    }
    __syncthreads();

    if (a.timers) { const long long t = clock64(); tm[0] += t - tprev; tprev = t; }
    // ---- row phase: upper row i = i0 + r*HS + tid, diagonals (x-r)*D + [0, D)
    const uint32_t* prev_cur = prevbuf + buf * H;   // iteration x-1's warp NW-1 words
    uint32_t* prev_next = prevbuf + (buf ^ 1) * H;
    // two slots per pass: their run chains are independent (ILP)
    constexpr int PR = (R % 2 == 0) ? 2 : 1;
#pragma unroll 1
    for (int r0 = 0; r0 < R; r0 += PR) {
      int lr[PR], rem[PR];
      RunState rs[PR];
      bool any_rem = false, all_full = true;
#pragma unroll
      for (int p = 0; p < PR; ++p) {
        const int r = r0 + p;
        lr[p] = r * HS + tid;
        prev_next[lr[p]] = rowbuf[(NW - 1) * H + lr[p]];
        const bool act = x >= r && lr[p] < hrows;
        rem[p] = act ? nrem - lr[p] - (x - r) * D : 0;  // valid diagonals of this row from k0
        any_rem |= rem[p] > 0;
        all_full &= rem[p] >= D;
      }
      if (!(a.skip & 2) && __any_sync(0xffffffffu, any_rem)) {
#pragma unroll
        for (int p = 0; p < PR; ++p) {
          const uint2 rsv = rowst[lr[p]];
          rs[p] = RunState{rsv.x, rsv.y};
        }
        if (__all_sync(0xffffffffu, all_full)) {          // common case: full words
#pragma unroll 2
          for (int v = 0; v < NW; ++v) {
#pragma unroll
            for (int p = 0; p < PR; ++p) {
              const uint32_t w = rowbuf[v * H + lr[p]];
              pts += __popc(w);
              runs_push(w, 32, rs[p], 0u, evq);
            }
            if (evq.tail - evq.head >= 32u) queue_drain(evq, hist, lane, false);
          }
        } else {
#pragma unroll 1
          for (int v = 0; v < NW; ++v) {
#pragma unroll
            for (int p = 0; p < PR; ++p) {
              const int nb = min(max(rem[p] - 32 * v, 0), 32);
              const uint32_t w = rowbuf[v * H + lr[p]] & low_mask(nb);
              pts += __popc(w);
              runs_push(w, nb, rs[p], 0u, evq);
            }
            if (evq.tail - evq.head >= 32u) queue_drain(evq, hist, lane, false);
          }
        }
#pragma unroll
        for (int p = 0; p < PR; ++p) {
          const int r = r0 + p;
          if (rem[p] > 0) {
            if (x == r) pts64 -= (rowbuf[lr[p]] & 1u);   // the diagonal cell counts once
            if (rem[p] <= D) {                             // the row ends at column n-1
              const Seg sg = runs_finish(rs[p]);
              lead_out[lr[p]] = sg.first;
              if (!sg.uniform) emit_run(sg.last, hist);
            }
          }
          rowst[lr[p]] = make_uint2(rs[p].first, rs[p].cur);
        }
      }
    }
    pts64 += 2ull * pts;
    pts = 0;
    if (a.timers) { const long long t = clock64(); tm[1] += t - tprev; tprev = t; }

    // ---- column phase: warp wv finishes column block u = wv (chunks wv..0)
    // and starts block u = wv + NW (chunks NW-1..wv+1) of every slot; lane =
    // column; rows are consumed bottom-up; two slots per pass (ILP).
    {
      Seg acc{0u, 0u, 0u};
      const int cfin = kx + 32 * wv + lane;      // finishing column, relative to i0
      const int cnew = cfin + D;                  // starting column
#pragma unroll 1
      for (int rr0 = 0; rr0 < R; rr0 += PR) {
        int rs_[PR], lim_fin[PR], lim_new[PR];
        RunState cur[PR], nst[PR], fin[PR];
#pragma unroll
        for (int p = 0; p < PR; ++p) {
          const int r = R - 1 - (rr0 + p);        // bottom-up over slots
          rs_[p] = r;
          const uint2 cs = colst[(wv * R + r) * 32 + lane];
          fin[p] = RunState{cs.y, cs.x};
          nst[p] = RunState{0u, 0u};
          cur[p] = RunState{0u, 0u};
          // rows of slot r above each column (relative to the slot's first row)
          lim_fin[p] = (x >= r && cfin < nrem) ? min(cfin, hrows) - r * HS : 0;
          lim_new[p] = (x >= r && cnew < nrem) ? min(cnew, hrows) - r * HS : 0;
        }
        if (!(a.skip & 4) && x >= rs_[PR - 1]) {   // the lower slot index is active last
#pragma unroll 1
          for (int c = NCH - 1; c >= 0; --c) {
            if (c == wv) {                          // switch to the finishing columns
#pragma unroll
              for (int p = 0; p < PR; ++p) {
                nst[p] = cur[p];
                cur[p] = fin[p];
              }
            }
            const bool finishing = c <= wv;
            const int wp = (wv - c) & (NW - 1);
#pragma unroll
            for (int p = 0; p < PR; ++p) {
              const int lr = rs_[p] * HS + 32 * c + lane;
              const uint32_t w1 = rowbuf[wp * H + lr];
              const uint32_t w0 = wp > 0 ? rowbuf[(wp - 1) * H + lr] : prev_cur[lr];
              const uint32_t colw = tr(__funnelshift_l(w0, w1, lane));
              const int nb = min(max((finishing ? lim_fin[p] : lim_new[p]) - 32 * c, 0), 32);
              const uint32_t bits = __funnelshift_rc(__brev(colw), 0u, 32 - nb);
              runs_push(bits, nb, cur[p], 0u, evq);
            }
            if (evq.tail - evq.head >= 32u) queue_drain(evq, hist, lane, false);
          }
#pragma unroll
          for (int p = 0; p < PR; ++p) fin[p] = cur[p];
        }
#pragma unroll
        for (int p = 0; p < PR; ++p) {
          acc = seg_combine(acc, runs_finish(fin[p]), hist);
          colst[(wv * R + rs_[p]) * 32 + lane] = make_uint2(nst[p].cur, nst[p].first);
        }
      }
      if (cfin < nrem) {
        // column part of hook (i0 + cfin) inside this band: rows [i0, min(i_end, i0 + cfin))
        Cb[cfin] = (cfin == 0) ? 0u
                 : acc.uniform ? pack_col(acc.first, acc.first)
                               : pack_col(acc.last, acc.first);  // (top, bottom)
      }
    }
    __syncthreads();

    if (a.timers) { const long long t = clock64(); tm[2] += t - tprev; tprev = t; }
    // ---- slot R-1 leaves the band through its bottom edge
    {
      const int kd = kx - (R - 1) * HS + delta;
      if (kd >= 0 && kd < nrem && kd < bot_rows)
        diag_finish(st[R - 1], true, Pb + kd, Sb + kd, LineSink{&hist, kd == 0 ? 1u : 2u});
    }
    if (((x + 1) & 4095) == 0) {
      for (int q = tid; q < 3 * kSmemBins; q += NW * 32) {
        const uint32_t cnt = sh_hist[q];
        if (cnt) {
          atomicAdd(&a.hist[(q / kSmemBins) * (n + 1) + (q % kSmemBins)], (unsigned long long)cnt);
          sh_hist[q] = 0u;
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int r = R - 1; r >= 1; --r) {
      st[r] = st[r - 1];
      if constexpr (!kDirect && kW > 0) {
        if constexpr (kLinfAnd) {
          ph_lo[r] = ph_lo[r - 1];
        } else {
#pragma unroll
          for (int j = 0; j < kW; ++j) win[r][j] = win[r - 1][j];
        }
      }
    }
  }

  // ---- drain: slots still holding diagonals after the last iteration.  All
  // their remaining cells lie right of column n-1: a segment with rows left
  // in the band is cut there; otherwise it leaves through the bottom edge.
#pragma unroll
  for (int dstep = 1; dstep < R; ++dstep) {
    const int kx = (X + dstep - 1) * D;
#pragma unroll
    for (int r = 1; r < R; ++r) {
      if (r >= dstep) {
        const int kd = kx - r * HS + delta;
        if (kd >= 0 && kd < nrem && hrows > r * HS && st[r].cur != 0u) {
          diag_finish(st[r], false, Pb + kd, Sb + kd, LineSink{&hist, kd == 0 ? 1u : 2u});
          st[r] = RunState{1u, 0u};  // finished: nothing left to report
        }
      }
    }
    {
      const int kd = kx - (R - 1) * HS + delta;
      if (kd >= 0 && kd < nrem && kd < bot_rows && st[R - 1].cur != 0u)
        diag_finish(st[R - 1], true, Pb + kd, Sb + kd, LineSink{&hist, kd == 0 ? 1u : 2u});
    }
#pragma unroll
    for (int r = R - 1; r >= 1; --r) st[r] = st[r - 1];
    st[0] = RunState{0u, 0u};
  }

  queue_drain(evq, hist, lane, true);
  if (a.timers && lane == 0) {
    const long long t = clock64();
    tm[3] += t - tprev;
    for (int k = 0; k < 4; ++k) atomicAdd(&a.timers[k], tm[k]);
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) pts64 += __shfl_xor_sync(0xffffffffu, pts64, o);
  if (lane == 0 && pts64) atomicAdd(a.points, pts64);
  __syncthreads();
  for (int q = tid; q < 3 * kSmemBins; q += NW * 32) {
    const uint32_t cnt = sh_hist[q];
    if (cnt) atomicAdd(&a.hist[(q / kSmemBins) * (n + 1) + (q % kSmemBins)], (unsigned long long)cnt);
  }
}

}  // namespace rqa
