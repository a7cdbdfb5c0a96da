// rqa_runs.cuh -- run-length monoid used to stitch vertical / white-vertical
// lines (runs of 1s / 0s) and diagonal lines across segment boundaries.
//
// A segment of a sequence is summarised by its first and last maximal runs
// (bit, length) along the traversal direction plus a "uniform" flag (the
// whole segment is one run); runs touching neither end are counted where
// they are found.  Combining consecutive segments is the reference's
// carry-over rule (engine.py:287-319) made associative, and emitting the
// end runs at the matrix border is flush_carryovers (engine.py:195-212).
#pragma once
#include "rqa_device.cuh"

namespace rqa {

// Run packed as (len << 1) | bit, len < 2^31.  len == 0: no run.
__host__ __device__ __forceinline__ uint32_t run_pack(uint32_t len, uint32_t bit) {
  return (len << 1) | bit;
}
__host__ __device__ __forceinline__ uint32_t run_len(uint32_t r) { return r >> 1; }
__host__ __device__ __forceinline__ uint32_t run_bit(uint32_t r) { return r & 1u; }

struct Seg {
  uint32_t first, last;  // packed runs; first == 0 means empty segment
  uint32_t uniform;      // 1: first == last and it covers the segment
};

template <class HistT>
__device__ __forceinline__ void emit_run(uint32_t r, const HistT& h) {
  const uint32_t len = run_len(r);
  if (len) h.add(run_bit(r) ? kVert : kWhite, len, 1u);
}

// a followed by b along the traversal direction.
template <class HistT>
__device__ __forceinline__ Seg seg_combine(Seg a, Seg b, const HistT& h) {
  if (a.first == 0u) return b;
  if (b.first == 0u) return a;
  const uint32_t al = a.last, bf = b.first;
  Seg r;
  if (run_bit(al) == run_bit(bf)) {
    const uint32_t m = run_pack(run_len(al) + run_len(bf), run_bit(al));
    if (a.uniform && b.uniform) return Seg{m, m, 1u};
    r.first = a.uniform ? m : a.first;
    r.last = b.uniform ? m : b.last;
    if (!a.uniform && !b.uniform) emit_run(m, h);
  } else {
    r.first = a.first;
    r.last = b.last;
    if (!a.uniform) emit_run(al, h);
    if (!b.uniform) emit_run(bf, h);
  }
  r.uniform = 0u;
  return r;
}

// Emit every run of a segment that touches a matrix border at both ends.
template <class HistT>
__device__ __forceinline__ void seg_flush(Seg s, const HistT& h) {
  if (s.first == 0u) return;
  emit_run(s.first, h);
  if (!s.uniform) emit_run(s.last, h);
}

// Streaming state of one sequence traversed bit by bit: `first` is the first
// run (0 while it is still open), `cur` the open run.  Interior runs are
// emitted as soon as they close.
struct RunState {
  uint32_t first, cur;
};

// Where closed runs go: vertical/white-vertical lines (both bit values) or
// diagonal lines (only runs of ones, with weight 2 for k > 0 by symmetry).
struct LineSink {
  const Hist* h;
  uint32_t diag_weight;  // 0: row/column sink; 1 or 2: diagonal sink
  __device__ __forceinline__ void operator()(uint32_t run) const {
    const uint32_t len = run_len(run);
    if (diag_weight == 0u) {
      h->add(run_bit(run) ? kVert : kWhite, len, 1u);
    } else if (run_bit(run)) {
      h->add(kDiag, len, diag_weight);
    }
  }
};

// Consume nb (1..32) bits of x, bit 0 first.  Run boundaries are the set
// bits of x ^ (x << 1 | carried bit); each one closes the open run.
__device__ __forceinline__ void runs_consume(uint32_t x, int nb, RunState& st, const LineSink& sink) {
  const uint32_t full = low_mask(nb);
  x &= full;
  uint32_t cur = st.cur;
  if (cur == 0u) cur = x & 1u;                         // sequence starts here
  uint32_t bnd = (x ^ ((x << 1) | (cur & 1u))) & full;
  if (bnd == 0u) {                                     // fast path: no boundary
    st.cur = cur + ((uint32_t)nb << 1);
    return;
  }
  uint32_t pos = 0;
  do {
    const uint32_t p = (uint32_t)__ffs(bnd) - 1u;
    const uint32_t run = cur + ((p - pos) << 1);
    if (st.first == 0u) st.first = run;
    else sink(run);
    cur = (cur & 1u) ^ 1u;
    pos = p;
    bnd &= bnd - 1u;
  } while (bnd);
  st.cur = cur + (((uint32_t)nb - pos) << 1);
}

// ---------------------------------------------------------------------------
// Deferred run emission.  A pass over one 64-bit word (two 32-bit words of a
// sequence) per lane only updates the lane's run state (branch-free); the
// runs the word closes are described by an event (64-bit boundary mask + the
// carried run) pushed into a per-warp ring in shared memory, and events are
// expanded 32 at a time, one per lane, so the histogram updates run at full
// SIMD width even when only a few lanes of a pass see a boundary.
// ---------------------------------------------------------------------------
constexpr int kQueueCap = 128;  // events per warp (16 bytes each)
// Drain when this many events are queued: every check follows at most 64
// pushes (two 64-bit words per lane), so the ring never holds more than 127.
#ifndef RQA_DRAIN_AT
#define RQA_DRAIN_AT 64u
#endif
constexpr uint32_t kDrainAt = RQA_DRAIN_AT;

// Event (16 bytes): x, y = boundary mask (bits 0..31, 32..63), z = carried
// run (len << 1 | bit) in bits 0..28 plus flags in bits 29..31: bit 29 skip
// the carried run (it is the sequence's first run, kept in the state), bits
// 30..31 diagonal weight (0: vertical/white sink).  Runs are shorter than 2^28
// (validate() bounds n).
constexpr uint32_t kEvCurBits = 29;
constexpr uint32_t kEvCurMask = (1u << kEvCurBits) - 1u;
// Shared word just past the histogram bins and the kernel's two mbarriers
// (SymSmem reserves it): the target of the zero-weight / out-of-range adds.
constexpr uint32_t kDummyBin = 3u * kSmemBins + 4u;

__device__ __forceinline__ void hist_red(const Hist& h, uint32_t kind_row, uint32_t len,
                                         uint32_t w) {
  // len < kSmemBins: 32-bit shared bin, unconditionally (a zero weight adds 0),
  // so ptxas emits no branch around it; longer lines go to the 64-bit global
  // counter in a rarely taken branch (the shared add then hits a dummy word)
  const bool small = len < (uint32_t)kSmemBins;
  const uint32_t sa = h.sh + 4u * (small ? kind_row * (uint32_t)kSmemBins + len : kDummyBin);
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(sa), "r"(small ? w : 0u) : "memory");
  if (!small && w) {
    RQA_DCHECK_AT(2, (int64_t)len < h.stride && kind_row < 3u);
    atomicAdd(h.g + (int64_t)kind_row * h.stride + len, (unsigned long long)w);
  }
}

__device__ __forceinline__ void expand_event(uint4 e, const Hist& h) {
  unsigned long long bnd = ((unsigned long long)e.y << 32) | e.x;
  const uint32_t flags = e.z >> kEvCurBits;
  const uint32_t w = flags >> 1;
  const uint32_t ecur = e.z & kEvCurMask;
  // weight and histogram row of runs of zeroes / ones
  const uint32_t w0 = (w == 0u) ? 1u : 0u, w1 = (w == 0u) ? 1u : w;
  const uint32_t k0 = kWhite, k1 = (w == 0u) ? (uint32_t)kVert : (uint32_t)kDiag;
  uint32_t bit = ecur & 1u;
  // first closed run: carried length + first boundary position
  uint32_t p = (uint32_t)__ffsll((long long)bnd) - 1u;
  uint32_t len = (ecur >> 1) + p;
  uint32_t wt = (flags & 1u) ? 0u : (bit ? w1 : w0);
  bnd &= bnd - 1ull;
  // two runs per trip: the second run's boundary scan does not wait for the
  // first run's histogram add (more independent work per lane)
  for (;;) {
    hist_red(h, bit ? k1 : k0, len, wt);  // wt == 0: predicated off
    if (bnd == 0ull) break;
    const uint32_t q1 = (uint32_t)__ffsll((long long)bnd) - 1u;
    const unsigned long long b2 = bnd & (bnd - 1ull);
    const uint32_t bit1 = bit ^ 1u;
    hist_red(h, bit1 ? k1 : k0, q1 - p, bit1 ? w1 : w0);
    if (b2 == 0ull) break;
    const uint32_t q2 = (uint32_t)__ffsll((long long)b2) - 1u;
    len = q2 - q1;
    p = q2;
    bnd = b2 & (b2 - 1ull);
    bit = bit1 ^ 1u;
    wt = bit ? w1 : w0;
  }
}

struct EventQueue {
  uint4* ring;       // this warp's kQueueCap entries
  uint32_t head;     // warp-uniform
  uint32_t tail;     // warp-uniform
  uint32_t lt_mask;  // (1 << lane) - 1
  uint32_t ring_sa;  // shared-window address of ring (set by the kernel)
};

// Expand whole groups of 32 events (all = true: everything left).  Kept out
// of line: it runs once per few passes and would otherwise be inlined at
// every pass site.
static __device__ __noinline__ uint32_t queue_drain_impl(uint32_t ring_sa, uint32_t head,
                                                         uint32_t tail, uint32_t sh,
                                                         unsigned long long* g, int64_t stride,
                                                         int lane, bool all) {
  const Hist h{sh, g, stride};
  while (tail - head >= 32u || (all && tail != head)) {
    const uint32_t avail = tail - head;
    if ((uint32_t)lane < avail) {
      uint4 e;
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(e.x), "=r"(e.y), "=r"(e.z), "=r"(e.w)
                   : "r"(ring_sa + 16u * ((head + lane) & (uint32_t)(kQueueCap - 1)))
                   : "memory");
      expand_event(e, h);
    }
    head += avail < 32u ? avail : 32u;
  }
  __syncwarp();
  return head;
}

__device__ __forceinline__ void queue_drain(EventQueue& q, const Hist& h, int lane, bool all) {
  __syncwarp();
  q.head = queue_drain_impl(q.ring_sa, q.head, q.tail, h.sh, h.g, h.stride, lane, all);
}

__device__ __forceinline__ void queue_check(EventQueue& q, const Hist& h, int lane) {
  if (q.tail - q.head >= kDrainAt) queue_drain(q, h, lane, false);
}

// One pass: consume nb (0..64) bits of lo | hi << 32, bit 0 first, into the
// lane's run state; closed runs go to the queue (no drain: the caller drains
// after at most two passes).  diag_weight 0: both run values count (vertical /
// white vertical); 1 or 2: only runs of ones count as diagonal lines with
// that weight.  All lanes of the warp must call it (nb = 0 for lanes with
// nothing to consume).  Branch-free.
__device__ __forceinline__ void runs_push(uint32_t lo, uint32_t hi, int nb, RunState& st,
                                          uint32_t diag_weight, EventQueue& q) {
  const uint32_t flo = (nb >= 32) ? 0xffffffffu : ((1u << nb) - 1u);
  const uint32_t fhi = (nb >= 64) ? 0xffffffffu : (nb > 32 ? ((1u << (nb - 32)) - 1u) : 0u);
  lo &= flo;
  hi &= fhi;
  const uint32_t cur = st.cur ? st.cur : (lo & 1u);                   // sequence starts here
  const uint32_t blo = (lo ^ ((lo << 1) | (cur & 1u))) & flo;          // run boundaries
  const uint32_t bhi = (hi ^ __funnelshift_l(lo, hi, 1)) & fhi;
  const bool ev = (blo | bhi) != 0u;
  const uint32_t plast = bhi ? 63u - (uint32_t)__clz(bhi) : 31u - (uint32_t)__clz(blo);
  const uint32_t p1 = blo ? (uint32_t)__ffs(blo) - 1u : 31u + (uint32_t)__ffs(bhi);
  // the last run's bit is the last consumed bit
  const uint32_t lastbit = (nb > 32 ? hi >> ((uint32_t)(nb - 33) & 31u) : lo >> ((uint32_t)(nb - 1) & 31u)) & 1u;
  const bool mkfirst = ev && st.first == 0u;                          // carried run is the first run
  const uint32_t cur_ev = (((uint32_t)nb - plast) << 1) | lastbit;
  st.first = mkfirst ? cur + (p1 << 1) : st.first;
  st.cur = ev ? cur_ev : cur + ((uint32_t)nb << 1);
  const uint32_t m = __ballot_sync(0xffffffffu, ev);
  // predicated store through a 32-bit shared address: no divergent branch and
  // no generic-address rematerialisation per push
  const uint32_t slot = (q.tail + __popc(m & q.lt_mask)) & (uint32_t)(kQueueCap - 1);
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@p st.shared.v4.u32 [%0], {%1, %2, %3, %3};\n\t}" ::"r"(q.ring_sa + 16u * slot),
      "r"(blo), "r"(bhi), "r"(cur | (((diag_weight << 1) | (mkfirst ? 1u : 0u)) << kEvCurBits)),
      "r"(ev ? 1u : 0u)
      : "memory");
  q.tail += __popc(m);
  RQA_DCHECK_AT(4, q.tail - q.head <= (uint32_t)kQueueCap);  // ring never overwrites unread events
}

__device__ __forceinline__ Seg runs_finish(const RunState& st) {
  if (st.cur == 0u) return Seg{0u, 0u, 0u};
  if (st.first == 0u) return Seg{st.cur, st.cur, 1u};
  return Seg{st.first, st.cur, 0u};
}

}  // namespace rqa
