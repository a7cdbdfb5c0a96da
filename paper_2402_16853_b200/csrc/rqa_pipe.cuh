// rqa_pipe.cuh -- software-pipelined upper-triangle band kernel.
//
// Same geometry, outputs and exactness rules as sym_kernel (rqa_sym.cuh), but
// the integer bookkeeping is interleaved with the FP64 work inside one
// instruction stream: the body of chunk c of iteration x holds
//   * the 32 FP64 steps of chunk c (R cells per lane per step),
//   * the diagonal runs + row-word transpose of chunk c-1 of iteration x,
//   * slice c of iteration x-1's row phase (word c of every slot's row) and
//     column phase (chunk NCH-1-c of every slot),
// all branch-free, so the FP64 pipe (cell test) and the ALU pipe (runs) work
// concurrently instead of alternating phase by phase.  Row words are
// double-buffered per iteration; one CTA barrier per iteration.
#pragma once
#include "rqa_sym.cuh"

namespace rqa {

constexpr int kPipeQueueCap = 256;  // events per warp: a chunk body pushes <= 3*R*32

struct PipeSmem {
  int H, HS, D, W, CW;
  size_t off_row, off_col0, off_col1, off_rowbuf0, off_rowbuf1, off_prev, off_colst, off_queue,
      off_hist, total;
  __host__ __device__ PipeSmem(int NW, int R, int W_) {
    D = 32 * NW;
    HS = D;
    H = R * HS;
    W = W_;
    CW = ((HS + D + W + 2) + 1) & ~1;
    off_row = 0;
    const size_t row_elems = ((size_t)(H + W) + 2) & ~(size_t)1;
    off_col0 = off_row + row_elems * sizeof(double);
    off_col1 = off_col0 + (size_t)CW * sizeof(double);
    off_rowbuf0 = off_col1 + (size_t)CW * sizeof(double);
    off_rowbuf1 = off_rowbuf0 + (size_t)NW * H * sizeof(uint32_t);
    off_prev = off_rowbuf1 + (size_t)NW * H * sizeof(uint32_t);
    off_colst = off_prev + 2 * (size_t)H * sizeof(uint32_t);
    off_queue = off_colst + (size_t)NW * R * 32 * sizeof(uint2);
    off_hist = off_queue + (size_t)NW * kPipeQueueCap * sizeof(uint4);
    total = off_hist + 3 * kSmemBins * sizeof(uint32_t) + 16;
  }
};

// Queue helpers for the larger ring.
__device__ __forceinline__ void pipe_push(uint32_t x, int nb, RunState& st, uint32_t diag_weight,
                                          uint4* ring, uint32_t& tail, uint32_t lt_mask) {
  const uint32_t full = (nb >= 32) ? 0xffffffffu : ((1u << nb) - 1u);
  x &= full;
  const uint32_t cur = st.cur ? st.cur : (x & 1u);
  const uint32_t bnd = (x ^ ((x << 1) | (cur & 1u))) & full;
  const bool ev = bnd != 0u;
  const uint32_t plast = 31u - (uint32_t)__clz(bnd);
  const uint32_t low = bnd & (0u - bnd);                       // lowest boundary bit
  const uint32_t p1 = 31u - (uint32_t)__clz(low);
  const bool mkfirst = ev && st.first == 0u;
  const uint32_t cur_ev = (((uint32_t)nb - plast) << 1) | ((x >> (plast & 31u)) & 1u);
  st.first = mkfirst ? cur + (p1 << 1) : st.first;
  st.cur = ev ? cur_ev : cur + ((uint32_t)nb << 1);
  const uint32_t m = __ballot_sync(0xffffffffu, ev);
  if (ev)
    ring[(tail + __popc(m & lt_mask)) % kPipeQueueCap] =
        make_uint4(bnd, cur, (diag_weight << 1) | (mkfirst ? 1u : 0u), 0u);
  tail += __popc(m);
}

static __device__ __noinline__ uint32_t pipe_drain_impl(const uint4* ring, uint32_t head,
                                                        uint32_t tail, uint32_t sh,
                                                        unsigned long long* g, int64_t stride,
                                                        int lane, bool all) {
  const Hist h{sh, g, stride};
  while (tail - head >= 32u || (all && tail != head)) {
    const uint32_t avail = tail - head;
    if ((uint32_t)lane < avail) expand_event(ring[(head + lane) % kPipeQueueCap], h);
    head += avail < 32u ? avail : 32u;
  }
  __syncwarp();
  return head;
}

template <int METRIC, int M, int TAU, int NW, int R, int MINB>
__global__ void __launch_bounds__(NW * 32, MINB)
pipe_kernel(const SymArgs a, const int W_rt) {
  constexpr int D = 32 * NW;
  constexpr int HS = D;
  constexpr int H = R * HS;
  constexpr bool kDirect = (M == 0);
  constexpr int kW = kDirect ? 0 : (M - 1) * TAU;
  constexpr bool kLinfAnd = (METRIC == kLinf) && (M >= 2);
  constexpr bool kSquare = (METRIC == kL2) && (M >= 2);
  constexpr int NCH = HS / 32;  // == NW: chunks per iteration == words per row per iteration
  static_assert(kLinfAnd ? kW <= 32 : kW <= 48, "term window too large");
  const int W = kDirect ? W_rt : kW;
  const PipeSmem L(NW, R, W);

  extern __shared__ __align__(128) unsigned char smem[];
  double* s_row = reinterpret_cast<double*>(smem + L.off_row);
  uint32_t* rowbufs[2] = {reinterpret_cast<uint32_t*>(smem + L.off_rowbuf0),
                          reinterpret_cast<uint32_t*>(smem + L.off_rowbuf1)};
  uint32_t* prevbuf = reinterpret_cast<uint32_t*>(smem + L.off_prev);
  uint2* colst = reinterpret_cast<uint2*>(smem + L.off_colst);
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
  const int nrem = (int)(n - i0);
  const int X = (nrem + D - 1) / D + R - 1;
  const int hrows = (int)(i_end - i0);
  const int bot_rows = (int)(n - i_end) + 1;
  const int theiler = (int)min(a.theiler, (int64_t)1 << 30);
  const double thr = a.thr;
  const int64_t boff = band_offset(b, n, a.row_lo, H);
  uint16_t* Pb = a.P + boff;
  uint16_t* Sb = a.S + boff;
  uint32_t* Cb = a.colsum + boff;
  uint32_t* lead_out = a.rowlead + i0;
  const Hist hist{smem_u32(sh_hist), a.hist, n + 1};
  const Transposer tr(lane);
  uint4* ring = reinterpret_cast<uint4*>(smem + L.off_queue) + wv * kPipeQueueCap;
  uint32_t qhead = 0u, qtail = 0u;
  const uint32_t lt_mask = (1u << lane) - 1u;
  auto drain = [&](bool all) {
    if (all || qtail - qhead >= 32u) {
      __syncwarp();
      qhead = pipe_drain_impl(ring, qhead, qtail, hist.sh, hist.g, hist.stride, lane, all);
    }
  };

  for (int q = tid; q < 3 * kSmemBins; q += NW * 32) sh_hist[q] = 0u;
  for (int q = tid; q < H + W; q += NW * 32) s_row[q] = a.s[i0 + q];
  for (int q = tid; q < 2 * H; q += NW * 32) prevbuf[q] = 0u;
  for (int q = tid; q < NW * R * 32; q += NW * 32) colst[q] = make_uint2(0u, 0u);
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

  RunState st[R];  // diagonal runs per slot (first run = band-top run)
  double win[R][kW > 0 ? kW : 1];
  uint32_t ph_lo[R], ph_hi[R];
  RunState rs[R];  // row part of hook (i0 + r*HS + tid)
#pragma unroll
  for (int r = 0; r < R; ++r) {
    st[r] = RunState{0u, 0u};
    rs[r] = RunState{0u, 0u};
    ph_lo[r] = 0u;
    ph_hi[r] = 0u;
  }
  uint32_t pts = 0;
  unsigned long long pts64 = 0;

  // -------------------------------------------------------------------------
  // previous-iteration (y = x - 1) row/column work, sliced over the chunks
  // -------------------------------------------------------------------------
  struct Slices {
    int rem[R];          // valid diagonals of row (r*HS + tid) from the start of iteration y
    RunState cur[R];     // column state being fed (starting, then finishing column)
    RunState nst[R];     // saved state of the starting column (lower part)
    RunState fin[R];     // state of the finishing column from iteration y-1
    int lim_fin[R], lim_new[R];
    int cfin;            // finishing column of this lane (relative to i0)
  } sl;
  auto slice_begin = [&](int y) {
    const int kx = y * D;
    sl.cfin = kx + 32 * wv + lane;
    const int cnew = sl.cfin + D;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int lr = r * HS + tid;
      const bool act = y >= r && lr < hrows;
      sl.rem[r] = act ? nrem - lr - (y - r) * D : 0;
      const uint2 cs = colst[(wv * R + r) * 32 + lane];
      sl.fin[r] = RunState{cs.y, cs.x};
      sl.nst[r] = RunState{0u, 0u};
      sl.cur[r] = RunState{0u, 0u};
      sl.lim_fin[r] = (y >= r && sl.cfin < nrem) ? min(sl.cfin, hrows) - r * HS : 0;
      sl.lim_new[r] = (y >= r && cnew < nrem) ? min(cnew, hrows) - r * HS : 0;
    }
  };
  // slice k of iteration y: word k of every row, column chunk NCH-1-k
  auto slice_step = [&](int y, int k, const uint32_t* rb, const uint32_t* prev, uint32_t* prev_next) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int lr = r * HS + tid;
      // row part: word k
      const int nb = min(max(sl.rem[r] - 32 * k, 0), 32);
      const uint32_t w = rb[k * H + lr] & low_mask(nb);
      pts += __popc(w);
      pipe_push(w, nb, rs[r], 0u, ring, qtail, lt_mask);
      if (k == NW - 1) prev_next[lr] = rb[(NW - 1) * H + lr];
      // column part: chunk cc, bottom-up
      const int cc = NCH - 1 - k;
      const bool sw = (cc == wv);  // switch from the starting to the finishing column
      sl.nst[r] = sw ? sl.cur[r] : sl.nst[r];
      sl.cur[r] = sw ? sl.fin[r] : sl.cur[r];
      const bool finishing = cc <= wv;
      const int wp = (wv - cc) & (NW - 1);
      const int clr = r * HS + 32 * cc + lane;
      const uint32_t w1 = rb[wp * H + clr];
      const uint32_t w0 = wp > 0 ? rb[(wp - 1) * H + clr] : prev[clr];
      const uint32_t colw = tr(__funnelshift_l(w0, w1, lane));
      const int cnb = min(max((finishing ? sl.lim_fin[r] : sl.lim_new[r]) - 32 * cc, 0), 32);
      const uint32_t bits = __funnelshift_rc(__brev(colw), 0u, 32 - cnb);
      pipe_push(bits, cnb, sl.cur[r], 0u, ring, qtail, lt_mask);
    }
  };
  auto slice_end = [&](int y) {
    Seg acc{0u, 0u, 0u};
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      const int r = R - 1 - rr;  // bottom-up over slots
      acc = seg_combine(acc, runs_finish(sl.cur[r]), hist);
      colst[(wv * R + r) * 32 + lane] = make_uint2(sl.nst[r].cur, sl.nst[r].first);
    }
    if (sl.cfin < nrem)
      Cb[sl.cfin] = (sl.cfin == 0) ? 0u
                  : acc.uniform ? pack_col(acc.first, acc.first)
                                : pack_col(acc.last, acc.first);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int lr = r * HS + tid;
      if (sl.rem[r] > 0) {
        if (y == r) pts64 -= (rowbufs[y & 1][lr] & 1u);  // the diagonal cell counts once
        if (sl.rem[r] <= D) {
          const Seg sg = runs_finish(rs[r]);
          lead_out[lr] = sg.first;
          if (!sg.uniform) emit_run(sg.last, hist);
        }
      }
    }
    pts64 += 2ull * pts;
    pts = 0;
  };

  for (int x = 0; x <= X; ++x) {
    const int kx = x * D;
    const int buf = x & 1;
    const bool have_prev = x > 0;       // iteration x-1's row/column work exists
    const bool compute = x < X;
    uint32_t* rb_cur = rowbufs[buf];
    const uint32_t* rb_prev = rowbufs[buf ^ 1];
    const uint32_t* prev_cur = prevbuf + (buf ^ 1) * H;   // words of iteration x-2 (for y = x-1)
    uint32_t* prev_next = prevbuf + buf * H;               // words of iteration x-1 (for y = x)
    if (have_prev) slice_begin(x - 1);

    if (compute) {
      if (tid == 0 && x + 1 < X) {
        const double* src;
        col_window_src(a.s, i0 + kx + D, &src);
        mbar_expect_tx_arrive(&bar[buf ^ 1], col_bytes);
        tma_load_1d(smem + (buf ? L.off_col0 : L.off_col1), src, col_bytes, &bar[buf ^ 1]);
      }
      mbar_wait(&bar[buf], (uint32_t)((x >> 1) & 1));
    }
    const int co = (int)((((uintptr_t)(a.s + i0 + kx)) >> 3) & 1);
    const double* s_col =
        reinterpret_cast<const double*>(smem + (buf ? L.off_col1 : L.off_col0)) + co + delta;

    int kdr[R], lastc[R], openb[R];
    if (compute) {
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
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int kd = kx - r * HS + delta;
      kdr[r] = kd;
      const int vrows = min(max(hrows - r * HS, 0), HS);
      const int crows = min(max(nrem - kd - r * HS, 0), vrows);
      lastc[r] = crows;
      openb[r] = (crows == vrows) ? 1 : 0;
    }

    // diagonal runs + row words of one finished chunk cc
    auto book = [&](int cc, const uint32_t (&words)[R], bool valid) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int kd = kdr[r];
        const bool live = valid && kd >= 0 && kd < nrem;
        const int rel = lastc[r] - 32 * cc;
        pipe_push(words[r], live ? min(max(rel, 0), 32) : 0, st[r], kd == 0 ? 1u : 2u, ring, qtail,
                  lt_mask);
        const uint32_t rw = tr(words[r]);
        if (valid) rb_cur[wv * H + r * HS + 32 * cc + lane] = rw;
      }
    };
    auto close_cut = [&](int cc) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int kd = kdr[r];
        const int rel = lastc[r] - 32 * cc;
        if (kd >= 0 && kd < nrem && !openb[r] && rel >= 0 && rel < 32 && st[r].cur != 0u) {
          diag_finish(st[r], false, Pb + kd, Sb + kd, LineSink{&hist, kd == 0 ? 1u : 2u});
          st[r] = RunState{1u, 0u};
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
      if (compute) {
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
      }
      // bookkeeping of chunk c-1 of this iteration and slice c of the previous
      book(c - 1, pw, compute && c > 0);
      if (have_prev) slice_step(x - 1, c, rb_prev, prev_cur, prev_next);
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
        pw[r] = (kdr[r] < theiler) ? 0u : word;
      }
      if (compute && c > 0) close_cut(c - 1);
      drain(false);
    }
    if (compute) {
      book(NCH - 1, pw, true);
      close_cut(NCH - 1);
    }
    if (have_prev) slice_end(x - 1);
    drain(false);
    __syncthreads();
    if (compute) {
      const int kd = kx - (R - 1) * HS + delta;
      if (kd >= 0 && kd < nrem && kd < bot_rows)
        diag_finish(st[R - 1], true, Pb + kd, Sb + kd, LineSink{&hist, kd == 0 ? 1u : 2u});
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
  }

  // ---- drain the diagonal slots after the last iteration (see sym_kernel)
#pragma unroll
  for (int dstep = 1; dstep < R; ++dstep) {
    const int kx = (X + dstep - 1) * D;
#pragma unroll
    for (int r = 1; r < R; ++r) {
      if (r >= dstep) {
        const int kd = kx - r * HS + delta;
        if (kd >= 0 && kd < nrem && hrows > r * HS && st[r].cur != 0u) {
          diag_finish(st[r], false, Pb + kd, Sb + kd, LineSink{&hist, kd == 0 ? 1u : 2u});
          st[r] = RunState{1u, 0u};
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

  drain(true);
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
