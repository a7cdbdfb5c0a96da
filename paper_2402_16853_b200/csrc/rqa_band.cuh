// rqa_band.cuh -- the fused tile kernel: neighbourhood test -> bit words ->
// diagonal / vertical / white-vertical run extraction -> histograms.
//
// Geometry.  One CTA owns a band of H = R*HS rows of the
// N x N recurrence matrix and sweeps it left to right in iterations of
// D = 32*NW diagonals.  Lane delta of warp v walks diagonal
//     k = k_x - r*HS + (32*v + lane)
// down the HS rows of slot r (r = 0..R-1) at iteration x.  All R slots of a
// lane touch the SAME column at a given step, so one shared-memory column
// load feeds R cells; slot r+1 at iteration x+1 continues slot r's diagonal
// from iteration x, so diagonal carries and the term window stay in
// registers (R>1 needs HS == D).
//
// Per cell the reference's arithmetic (embedding.py:137-156) is reproduced
// bit-exactly: d = s[row+k*tau] - s[col+k*tau]; L2 (m>1): d*d, L1 / m=1: |d|;
// accumulation in k order with IEEE adds (no FMA: -fmad=false and __d*_rn);
// sqrt removed via the exact threshold T* (SURVEY App. A.2); Linf as the AND
// of per-component predicates (App. A.3).  Terms are reused along the
// diagonal: component k of cell (i,j) is component 0 of (i+k*tau, j+k*tau)
// (App. A.4), so each cell costs one new sub(+mul) plus m-1 adds.
#pragma once
#include "rqa_device.cuh"

namespace rqa {

// Dynamic shared memory layout (bytes), identical on host and device.
struct BandSmem {
  int H, HS, D, W, CW;
  size_t off_row, off_col0, off_col1, off_rowbuf, off_hist, total;
  __host__ __device__ BandSmem(int NW, int R, int HS_, int W_) {
    HS = HS_;
    H = R * HS_;
    D = 32 * NW;
    W = W_;
    CW = ((HS + D + W + 2) + 1) & ~1;          // column window (+1 for alignment), even
    off_row = 0;
    size_t row_elems = ((size_t)(H + W) + 1) & ~(size_t)1;
    off_col0 = off_row + row_elems * sizeof(double);
    off_col1 = off_col0 + (size_t)CW * sizeof(double);
    off_rowbuf = off_col1 + (size_t)CW * sizeof(double);
    off_hist = off_rowbuf + (size_t)NW * H * sizeof(uint32_t);
    total = off_hist + 3 * kSmemBins * sizeof(uint32_t) + 16 /* two mbarriers */;
  }
};


__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx_arrive(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// 1-D TMA bulk copy global -> shared, completion counted on an mbarrier.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Stage s[i0+k_x+q] (q in [0, CW-1)) into a column buffer; returns the
// element offset introduced by aligning the source down to 16 bytes.
template <typename T>
__device__ __forceinline__ int col_window_src(const T* s, int64_t start, const T** src) {
  const uintptr_t a = (uintptr_t)(s + start);
  const int off = (int)((a & 15u) / sizeof(T));
  *src = s + start - off;
  return off;
}

template <int METRIC, int M, int TAU, int NW, int R, int HS>
struct BandCfg {
  static constexpr bool kDirect = (M == 0);                 // runtime m, tau (no term reuse)
  static constexpr int kW = kDirect ? 0 : (M - 1) * TAU;   // compile-time term window
  static constexpr int kD = 32 * NW;
  static constexpr int kH = R * HS;
  static constexpr bool kLinfAnd = (METRIC == kLinf) && (M >= 2);
  static constexpr bool kSquare = (METRIC == kL2) && (M >= 2);
  static_assert(HS % 32 == 0, "slot height must be a multiple of 32");
  static_assert(R == 1 || HS == kD, "stacked slots need HS == D");
  static_assert(kW <= 32, "term window too large for the reuse kernel");
};

template <int METRIC, int M, int TAU, int NW, int R, int HS>
__global__ void __launch_bounds__(NW * 32)
band_kernel(const BandArgs a, const int W_rt) {
  using C = BandCfg<METRIC, M, TAU, NW, R, HS>;
  constexpr int D = C::kD;
  constexpr int H = C::kH;
  constexpr int kW = C::kW;
  constexpr int NCH = HS / 32;
  const int W = C::kDirect ? W_rt : kW;
  const BandSmem L(NW, R, HS, W);

  extern __shared__ __align__(128) unsigned char smem[];
  double* s_row = reinterpret_cast<double*>(smem + L.off_row);
  double* s_colbuf[2] = {reinterpret_cast<double*>(smem + L.off_col0),
                         reinterpret_cast<double*>(smem + L.off_col1)};
  uint32_t* rowbuf = reinterpret_cast<uint32_t*>(smem + L.off_rowbuf);
  uint32_t* sh_hist = reinterpret_cast<uint32_t*>(smem + L.off_hist);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L.off_hist + 3 * kSmemBins * sizeof(uint32_t));

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int v = tid >> 5;
  const int delta = 32 * v + lane;
  const int64_t n = a.n;
  const int64_t i0 = a.row_lo + (int64_t)blockIdx.x * H;
  const int64_t i_end = min(i0 + (int64_t)H, a.row_hi);
  const int64_t kx0 = -(i0 + HS - 1);
  const int64_t X = (n + HS - 1 + D - 1) / D;
  const double thr = a.thr;
  uint16_t* Pb = a.P + (int64_t)blockIdx.x * n;
  uint16_t* Sb = a.S + (int64_t)blockIdx.x * n;
  const Hist hist{smem_u32(sh_hist), a.hist, n + 1};

  for (int q = tid; q < 3 * kSmemBins; q += NW * 32) sh_hist[q] = 0u;
  for (int q = tid; q < H + W; q += NW * 32) s_row[q] = a.s[i0 + q];
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // Column windows are double-buffered, one mbarrier per buffer: the load for
  // iteration x+1 is armed on bar[(x+1)&1], whose previous phase every thread
  // waited on during iteration x-1 (before that iteration's final barrier).
  const uint32_t col_bytes = (uint32_t)(L.CW * sizeof(double));
  if (tid == 0) {
    const double* src;
    col_window_src(a.s, i0 + kx0, &src);
    mbar_expect_tx_arrive(&bar[0], col_bytes);
    tma_load_1d(s_colbuf[0], src, col_bytes, &bar[0]);
  }

  // ---- per-lane slot state -------------------------------------------------
  DiagRun st[R];
  double win[R][kW > 0 ? kW : 1];
  uint32_t ph_lo[R], ph_hi[R];  // Linf: predicate bits (lookahead window)
#pragma unroll
  for (int r = 0; r < R; ++r) {
    st[r].len = 0;
    st[r].rooted = 0;
    ph_lo[r] = 0u;
    ph_hi[r] = 0u;
  }
  // rows owned by this thread in the row phase: lr = tid + q*D
  constexpr int RQ = H / D;
  RowRun rs[RQ];
#pragma unroll
  for (int q = 0; q < RQ; ++q) {
    rs[q].bit = -1;
    rs[q].len = 0;
  }
  unsigned long long pts = 0;

  for (int64_t x = 0; x < X; ++x) {
    const int64_t kx = kx0 + x * D;
    const int buf = (int)(x & 1);
    // prefetch the next iteration's column window (its buffer was released by
    // the barrier that ended iteration x-1)
    if (tid == 0 && x + 1 < X) {
      const double* src;
      col_window_src(a.s, i0 + kx + D, &src);
      mbar_expect_tx_arrive(&bar[buf ^ 1], col_bytes);
      tma_load_1d(s_colbuf[buf ^ 1], src, col_bytes, &bar[buf ^ 1]);
    }
    mbar_wait(&bar[buf], (uint32_t)((x >> 1) & 1));
    // same 16-byte alignment offset as col_window_src computed for this window
    const int co = (int)((((uintptr_t)(a.s + i0 + kx)) >> 3) & 1);
    const double* s_col = s_colbuf[buf] + co + delta;  // s_col[u] = s[i0 + kx + delta + u]

    // ---- warm-up of fresh slots: slot 0 always, every slot on the first pass
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (r == 0 || x == 0) {
        const int64_t kd = kx - (int64_t)r * HS + delta;
        st[r].len = 0;
        st[r].rooted = (r == 0 && kd >= 0 && kd < n && i0 + kd < n) ? 1 : 0;
        if constexpr (!C::kDirect && kW > 0) {
          if constexpr (C::kLinfAnd) {
            uint32_t p = 0;
#pragma unroll
            for (int u = 0; u < kW; ++u) {
              const double d = __dsub_rn(s_row[r * HS + u], s_col[u]);
              if (fabs(d) <= thr) p |= 1u << u;
            }
            ph_lo[r] = p;
            ph_hi[r] = 0u;
          } else {
#pragma unroll
            for (int u = 0; u < kW; ++u) {
              const double d = __dsub_rn(s_row[r * HS + u], s_col[u]);
              win[r][u] = C::kSquare ? __dmul_rn(d, d) : fabs(d);
            }
          }
        }
      }
    }

    for (int c = 0; c < NCH; ++c) {
      uint32_t dw[R];
#pragma unroll
      for (int r = 0; r < R; ++r) dw[r] = 0u;
      const double* colc = s_col + 32 * c;
      const double* rowc = s_row + 32 * c;
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        if constexpr (!C::kDirect) {
          const double cv = colc[t + kW];
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const double rv = rowc[r * HS + t + kW];
            const double d = __dsub_rn(rv, cv);
            if constexpr (M == 1) {
              if (fabs(d) <= thr) dw[r] |= 1u << t;
            } else if constexpr (C::kLinfAnd) {
              if (fabs(d) <= thr) {
                if (t + kW < 32) ph_lo[r] |= 1u << ((t + kW) & 31);
                else ph_hi[r] |= 1u << ((t + kW - 32) & 31);
              }
            } else {
              const double term = C::kSquare ? __dmul_rn(d, d) : fabs(d);
              double acc = win[r][0];
#pragma unroll
              for (int k = 1; k < M - 1; ++k) acc = __dadd_rn(acc, win[r][k * TAU]);
              acc = __dadd_rn(acc, term);
              if (acc <= thr) dw[r] |= 1u << t;
#pragma unroll
              for (int j = 0; j + 1 < kW; ++j) win[r][j] = win[r][j + 1];
              win[r][kW - 1] = term;
            }
          }
        } else {
          // direct evaluation with runtime m, tau (embedding.py:137-156 verbatim)
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

      // ---- per slot: diagonal runs, transpose, row words to shared memory
#pragma unroll
      for (int r = 0; r < R; ++r) {
        uint32_t word;
        if constexpr (C::kLinfAnd) {
          word = ph_lo[r];
#pragma unroll
          for (int k = 1; k < M; ++k) word &= __funnelshift_rc(ph_lo[r], ph_hi[r], k * TAU);
          ph_lo[r] = ph_hi[r];
          ph_hi[r] = 0u;
        } else {
          word = dw[r];
        }
        const int64_t kd = kx - (int64_t)r * HS + delta;
        const int64_t akd = kd < 0 ? -kd : kd;
        if (akd < a.theiler) word = 0u;
        if (kd >= 0 && kd < n) {
          const int64_t base = i0 + (int64_t)r * HS + 32 * c;
          const int64_t lb = imin64(imax64(i_end - base, 0), 32);
          const int64_t lcb = imin64(imax64(n - kd - base, 0), lb);
          diag_word(word, (int)lcb, (int)lb, st[r], Pb + kd, kd == 0 ? 1u : 2u, hist);
        }
        const uint32_t rw = transpose32(word, lane);
        rowbuf[v * H + r * HS + 32 * c + lane] = rw;
      }
    }
    __syncthreads();

    // ---- row phase: each thread owns rows lr = tid + q*D of the band
#pragma unroll
    for (int q = 0; q < RQ; ++q) {
      const int lr = tid + q * D;
      const int64_t gi = i0 + lr;
      if (gi < i_end) {
        const int64_t cb = i0 + (lr % HS) + kx;  // column of bit 0 of warp 0's word
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          const int64_t cs = cb + 32 * w;
          const int64_t lo = imax64(-cs, 0);
          const int64_t hi = imin64(n - cs, 32);
          if (hi > lo) {
            const uint32_t word = rowbuf[w * H + lr] >> lo;
            const int nb = (int)(hi - lo);
            pts += __popc(word & low_mask(nb));
            row_bits(word, nb, rs[q], hist);
          }
        }
      }
    }

    // ---- slot R-1 leaves the band through its bottom edge
    {
      const int64_t kd = kx - (int64_t)(R - 1) * HS + delta;
      if (kd >= 0 && kd < n && i_end - 1 + kd < n) {
        DiagRun& e = st[R - 1];
        if (e.rooted) Pb[kd] = (uint16_t)e.len;
        Sb[kd] = (uint16_t)e.len;
      }
    }
    // keep the 32-bit shared bins far from overflow on very long sweeps
    if (((x + 1) & 4095) == 0) {
      __syncthreads();
      for (int q = tid; q < 3 * kSmemBins; q += NW * 32) {
        const uint32_t cnt = sh_hist[q];
        if (cnt) {
          atomicAdd(&a.hist[(q / kSmemBins) * (n + 1) + (q % kSmemBins)], (unsigned long long)cnt);
          sh_hist[q] = 0u;
        }
      }
    }
    // rotate slots: slot r+1 continues slot r's diagonals next iteration
#pragma unroll
    for (int r = R - 1; r >= 1; --r) {
      st[r] = st[r - 1];
      if constexpr (!C::kDirect && kW > 0) {
        if constexpr (C::kLinfAnd) {
          ph_lo[r] = ph_lo[r - 1];
        } else {
#pragma unroll
          for (int j = 0; j < kW; ++j) win[r][j] = win[r - 1][j];
        }
      }
    }
    __syncthreads();
  }

  // ---- drain: slots still holding diagonals after the last iteration.  All
  // their remaining cells lie right of column n-1, so a run ends at the first
  // remaining row inside the band, or leaves through the bottom edge.
#pragma unroll
  for (int dstep = 1; dstep < R; ++dstep) {
    const int64_t kx = kx0 + (X + dstep - 1) * D;
#pragma unroll
    for (int r = 1; r < R; ++r) {
      if (r >= dstep) {
        const int64_t kd = kx - (int64_t)r * HS + delta;
        if (kd >= 0 && kd < n && i_end > i0 + (int64_t)r * HS && (st[r].len | st[r].rooted))
          diag_end_run(st[r], Pb + kd, kd == 0 ? 1u : 2u, hist);
      }
    }
    {
      const int64_t kd = kx - (int64_t)(R - 1) * HS + delta;
      if (kd >= 0 && kd < n && i_end - 1 + kd < n) {
        DiagRun& e = st[R - 1];
        if (e.rooted) Pb[kd] = (uint16_t)e.len;
        Sb[kd] = (uint16_t)e.len;
      }
    }
#pragma unroll
    for (int r = R - 1; r >= 1; --r) st[r] = st[r - 1];
    st[0].len = 0;
    st[0].rooted = 0;
  }

  // ---- rows end at column n-1: count the open runs (flush, engine.py:195-212)
#pragma unroll
  for (int q = 0; q < RQ; ++q) row_emit(rs[q], hist);

  // ---- points and shared histogram -> global
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) pts += __shfl_xor_sync(0xffffffffu, pts, o);
  if (lane == 0 && pts) atomicAdd(a.points, pts);
  __syncthreads();
  for (int q = tid; q < 3 * kSmemBins; q += NW * 32) {
    const uint32_t c = sh_hist[q];
    if (c) atomicAdd(&a.hist[(q / kSmemBins) * (n + 1) + (q % kSmemBins)], (unsigned long long)c);
  }
}

}  // namespace rqa
