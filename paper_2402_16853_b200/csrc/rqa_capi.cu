// rqa_capi.cu -- host side of librqa_b200.so: validation, exact threshold,
// device workspaces, kernel launches and the C-ABI of include/rqa_b200.h.
#include <algorithm>
#include <atomic>
#include <cfloat>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/rqa_b200.h"
#include "rqa_fold.cuh"
#include "rqa_variants.cuh"

namespace rqa {
namespace {

std::atomic<int64_t> g_launches{0};

void set_err(char* err, size_t errlen, const char* fmt, ...) {
  if (!err || errlen == 0) return;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(err, errlen, fmt, ap);
  va_end(ap);
}

// T* = max{x : RN(sqrt(x)) <= eps}; acc <= T*  <=>  sqrt(acc) <= eps for
// every acc >= +0 and for NaN.  Never eps*eps.
double l2_threshold(double eps) {
  if (std::isinf(eps)) return INFINITY;
  double t = eps * eps;
  if (std::isinf(t)) t = DBL_MAX;
  while (t > 0.0 && std::sqrt(t) > eps) t = std::nextafter(t, 0.0);
  for (;;) {
    const double u = std::nextafter(t, INFINITY);
    if (std::isinf(u) || std::sqrt(u) > eps) break;
    t = u;
  }
  return t;
}

double threshold_for(int metric, int m, double radius) {
  return (metric == kL2 && m > 1) ? l2_threshold(radius) : radius;
}

struct Workspace {
  std::mutex mu;
  cudaStream_t stream = nullptr;
  double* s_pad = nullptr;
  size_t s_cap = 0;  // elements
  uint16_t* ps = nullptr;      // P and S (compact band layout)
  size_t ps_cap = 0;  // elements
  uint32_t* cs = nullptr;      // column-part summaries (compact band layout)
  size_t cs_cap = 0;
  uint32_t* rowlead = nullptr; // [2n] row part per row (single-device final mode)
  size_t rowlead_cap = 0;
  uint2* rowpiece = nullptr;   // [nunits][H]
  size_t rowpiece_cap = 0;
  Unit* units = nullptr;       // [nunits] launch order
  size_t units_cap = 0;
  int4* units_bb = nullptr;    // [nunits] sorted by band, xa
  size_t units_bb_cap = 0;
  int32_t* band_start = nullptr;
  size_t band_start_cap = 0;
  int32_t* stripe_buf = nullptr;  // auto-striping: [G][n] x2 + [G][2n] + [2n]
  size_t stripe_buf_cap = 0;
  unsigned long long* hist = nullptr;
  size_t hist_cap = 0;  // elements (3*(n+1) + 1 for points)
  int64_t* bounds = nullptr;
  size_t bounds_cap = 0;
  cudaEvent_t ev[6] = {};
  bool init = false;
};

std::mutex g_ws_mu;
std::vector<Workspace*> g_ws;

Workspace* workspace(int dev) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  if ((int)g_ws.size() <= dev) g_ws.resize(dev + 1, nullptr);
  if (!g_ws[dev]) g_ws[dev] = new Workspace();
  return g_ws[dev];
}

template <typename T>
cudaError_t grow(T** p, size_t* cap, size_t need) {
  if (*cap >= need) return cudaSuccess;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), need * sizeof(T));
  if (e == cudaSuccess) *cap = need;
  return e;
}

struct Problem {
  int64_t len, n;
  int m, tau, metric;
  double radius, thr;
  int64_t theiler;
  Variant var;
  int64_t pad;  // zero padding on each side of the staged series
};

int validate(int64_t len, int32_t m, int32_t tau, int32_t metric, double radius,
             int64_t theiler, Problem* p, char* err, size_t errlen) {
  if (m < 1) return set_err(err, errlen, "embedding_dimension must be >= 1"), RQA_EINVAL;
  if (tau < 1) return set_err(err, errlen, "time_delay must be >= 1"), RQA_EINVAL;
  if (metric < 0 || metric > 2) return set_err(err, errlen, "unknown metric %d", metric), RQA_EINVAL;
  if (!(radius >= 0)) return set_err(err, errlen, "radius must be >= 0"), RQA_EINVAL;
  if (theiler < 0) return set_err(err, errlen, "theiler window must be >= 0"), RQA_EINVAL;
  const int64_t span = (int64_t)(m - 1) * tau;
  if (len <= span)
    return set_err(err, errlen,
                   "series of length %lld cannot be embedded with m=%d, tau=%d (needs more than "
                   "%lld samples)",
                   (long long)len, m, tau, (long long)span),
           RQA_ESHORT;
  p->len = len;
  p->n = len - span;
  if (p->n > (int64_t)1 << 31)
    return set_err(err, errlen, "n_vectors %lld exceeds 2^31", (long long)p->n), RQA_EINVAL;
  p->m = m;
  p->tau = tau;
  p->metric = metric;
  p->radius = radius;
  p->thr = threshold_for(metric, m, radius);
  p->theiler = theiler;
  if (!find_variant(metric, m, tau, p->n, &p->var))
    return set_err(err, errlen, "embedding window (m-1)*tau = %lld too large (max 4096)",
                   (long long)span),
           RQA_EINVAL;
  const int64_t H = p->var.band_rows(), D = 32 * p->var.nw;
  p->pad = 2 * H + 4 * D + p->var.w + 256;
  (void)D;
  return RQA_OK;
}

int cuda_fail(cudaError_t e, const char* what, char* err, size_t errlen) {
  set_err(err, errlen, "%s: %s", what, cudaGetErrorString(e));
  return e == cudaErrorMemoryAllocation ? RQA_ENOMEM : RQA_EDEVICE;
}

#define RQA_CUDA(call, what)                                  \
  do {                                                        \
    cudaError_t e_ = (call);                                  \
    if (e_ != cudaSuccess) return cuda_fail(e_, what, err, errlen); \
  } while (0)

// Stage the series into the zero-padded workspace buffer.
int stage_series(Workspace* ws, const Problem& p, const double* src, cudaMemcpyKind kind,
                 cudaStream_t st, char* err, size_t errlen) {
  const size_t need = (size_t)(p.len + 2 * p.pad);
  RQA_CUDA(grow(&ws->s_pad, &ws->s_cap, need), "allocating series buffer");
  RQA_CUDA(cudaMemsetAsync(ws->s_pad, 0, (size_t)p.pad * sizeof(double), st), "memset pad");
  RQA_CUDA(cudaMemsetAsync(ws->s_pad + p.pad + p.len, 0, (size_t)p.pad * sizeof(double), st),
           "memset pad");
  RQA_CUDA(cudaMemcpyAsync(ws->s_pad + p.pad, src, (size_t)p.len * sizeof(double), kind, st),
           "copying series");
  return RQA_OK;
}

// Work units: every band's diagonal sweep is cut into iteration ranges of
// about `len` iterations so that the grid has several waves of similar CTAs
// (the upper triangle makes the first bands the longest).
struct UnitPlan {
  std::vector<Unit> units;       // launch order (longest first)
  std::vector<int4> by_band;     // (band, xa, xb, idx) sorted by band, xa
  std::vector<int32_t> band_start;
};

UnitPlan plan_units(const Problem& p, int64_t row_lo, int64_t row_hi, int slots) {
  const int64_t H = p.var.band_rows(), D = p.var.slot_rows(), R = p.var.r;
  const int64_t nb = (row_hi - row_lo + H - 1) / H;
  std::vector<int64_t> X(nb);
  int64_t total = 0;
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t nrem = p.n - (row_lo + b * H);
    X[b] = (nrem + D - 1) / D + R - 1;
    total += X[b];
  }
  // aim for >= 4 waves of units; one recomputed iteration per unit boundary
  int64_t len = std::max<int64_t>(8, total / std::max<int64_t>(1, 4LL * slots));
  UnitPlan pl;
  pl.band_start.assign(nb + 1, 0);
  for (int64_t b = 0; b < nb; ++b) {
    pl.band_start[b] = (int32_t)pl.by_band.size();
    const int64_t parts = std::max<int64_t>(1, (X[b] + len - 1) / len);
    for (int64_t q = 0; q < parts; ++q) {
      const int32_t xa = (int32_t)(X[b] * q / parts), xb = (int32_t)(X[b] * (q + 1) / parts);
      const int32_t idx = (int32_t)pl.units.size();
      pl.units.push_back(Unit{(int32_t)b, xa, xb, idx});
      pl.by_band.push_back(make_int4((int)b, xa, xb, idx));
    }
  }
  pl.band_start[nb] = (int32_t)pl.by_band.size();
  std::stable_sort(pl.units.begin(), pl.units.end(),
                   [](const Unit& u, const Unit& v) { return (u.xb - u.xa) > (v.xb - v.xa); });
  return pl;
}

int64_t unit_workspace_bytes(const Problem& p, int64_t row_lo, int64_t row_hi) {
  const int64_t H = p.var.band_rows(), HS = p.var.slot_rows();
  const int64_t nb = (row_hi - row_lo + H - 1) / H;
  const int64_t nslots = (row_hi - row_lo + HS - 1) / HS;
  return 2 * slot_offset(nslots, p.n, row_lo, HS) * 2 + sym_band_offset(nb, p.n, row_lo, H) * 4;
}

// Work-unit kernel over rows [row_lo, row_hi) + folds.
//   final mode: diagonal and hook folds write the complete histograms;
//   stripe mode: per-stripe summaries for the cross-stripe stitch.
int launch_rows(Workspace* ws, const Problem& p, int64_t row_lo, int64_t row_hi, int mode,
                unsigned long long* hist, unsigned long long* points, int32_t* out_p,
                int32_t* out_s, uint32_t* out_col, uint32_t* out_row, cudaStream_t st,
                cudaEvent_t ev_mid, char* err, size_t errlen) {
  const int64_t H = p.var.band_rows(), HS = p.var.slot_rows();
  const int64_t nb = (row_hi - row_lo + H - 1) / H;
  if (nb <= 0) return RQA_OK;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  RQA_CUDA(cudaFuncSetAttribute(p.var.kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)p.var.smem),
           "kernel attributes");
  RQA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, p.var.kernel, 32 * p.var.nw,
                                                         p.var.smem),
           "occupancy");
  const UnitPlan pl = plan_units(p, row_lo, row_hi, sms * std::max(1, per_sm));
  const int64_t nunits = (int64_t)pl.units.size();
  const int64_t nslots = (row_hi - row_lo + HS - 1) / HS;
  const int64_t ptot = slot_offset(nslots, p.n, row_lo, HS);
  const int64_t ctot = sym_band_offset(nb, p.n, row_lo, H);
  RQA_CUDA(grow(&ws->ps, &ws->ps_cap, (size_t)(2 * ptot)), "allocating diagonal summaries");
  RQA_CUDA(grow(&ws->cs, &ws->cs_cap, (size_t)ctot), "allocating column summaries");
  RQA_CUDA(grow(&ws->rowpiece, &ws->rowpiece_cap, (size_t)(nunits * H)), "allocating row pieces");
  RQA_CUDA(grow(&ws->units, &ws->units_cap, (size_t)nunits), "allocating units");
  RQA_CUDA(grow(&ws->units_bb, &ws->units_bb_cap, (size_t)nunits), "allocating units");
  RQA_CUDA(grow(&ws->band_start, &ws->band_start_cap, (size_t)nb + 1), "allocating units");
  RQA_CUDA(cudaMemcpyAsync(ws->units, pl.units.data(), nunits * sizeof(Unit),
                           cudaMemcpyHostToDevice, st),
           "copying units");
  RQA_CUDA(cudaMemcpyAsync(ws->units_bb, pl.by_band.data(), nunits * sizeof(int4),
                           cudaMemcpyHostToDevice, st),
           "copying units");
  RQA_CUDA(cudaMemcpyAsync(ws->band_start, pl.band_start.data(), (nb + 1) * sizeof(int32_t),
                           cudaMemcpyHostToDevice, st),
           "copying units");
  uint32_t* rowpart = out_row;
  if (!rowpart) {  // final mode: the hook fold does not need a separate row-part array
    RQA_CUDA(grow(&ws->rowlead, &ws->rowlead_cap, (size_t)(2 * p.n)), "allocating row parts");
    rowpart = ws->rowlead;
  }

  UnitArgs ua;
  memset(&ua, 0, sizeof ua);
  SymArgs& a = ua.base;
  a.s = ws->s_pad + p.pad;
  a.len = p.len;
  a.n = p.n;
  a.row_lo = row_lo;
  a.row_hi = row_hi;
  a.thr = p.thr;
  a.theiler = p.theiler;
  a.m = p.m;
  a.tau = p.tau;
  a.P = ws->ps;               // [2][ptot]: P then S, per-slot compact layout
  a.S = ws->ps + ptot;
  a.colsum = ws->cs;
  a.rowlead = nullptr;
  a.hist = hist;
  a.points = points;
  static const char* skip_env = getenv("RQA_SKIP");  // profiling only: skip phases
  a.skip = skip_env ? atoi(skip_env) : 0;
  a.timers = nullptr;
  ua.units = ws->units;
  ua.rowpiece = ws->rowpiece;
  RQA_CUDA(p.var.launch(ua, (int)nunits, p.var.w, st), "launching band kernel");
  g_launches++;
  if (ev_mid) RQA_CUDA(cudaEventRecord(ev_mid, st), "event");

  const int threads = 256;
  const int64_t blocks = std::min<int64_t>((p.n + threads - 1) / threads, 148 * 16);
  SymFoldArgs f;
  memset(&f, 0, sizeof f);
  f.P = a.P;
  f.S = a.S;
  f.row_lo = row_lo;
  f.row_hi = row_hi;
  f.H = HS;                   // diagonal segments are slots
  f.nb = (int)nslots;
  f.n = p.n;
  f.hist = hist;
  f.out_p = out_p;
  f.out_s = out_s;
  sym_fold_diag<<<(int)blocks, threads, 0, st>>>(f, mode);
  RQA_CUDA(cudaGetLastError(), "launching diagonal fold");
  UnitFoldArgs h;
  memset(&h, 0, sizeof h);
  h.colsum = ws->cs;
  h.rowpiece = ws->rowpiece;
  h.units_by_band = ws->units_bb;
  h.band_start = ws->band_start;
  h.row_lo = row_lo;
  h.row_hi = row_hi;
  h.H = H;
  h.HS = HS;
  h.D = p.var.slot_rows();
  h.nb = (int)nb;
  h.n = p.n;
  h.hist = hist;
  h.out_col = reinterpret_cast<uint2*>(out_col);
  h.out_row = reinterpret_cast<uint2*>(rowpart);
  unit_fold_hooks<<<(int)blocks, threads, 0, st>>>(h, mode);
  RQA_CUDA(cudaGetLastError(), "launching hook fold");
  g_launches += 2;
  return RQA_OK;
}

int stitch_stripes(Workspace* ws, const int32_t* d_prefix, const int32_t* d_suffix,
                   const uint32_t* d_col, const uint32_t* d_row, const int64_t* bounds,
                   int32_t nstripes, int64_t n, unsigned long long* hist, cudaStream_t st,
                   char* err, size_t errlen) {
  RQA_CUDA(grow(&ws->bounds, &ws->bounds_cap, (size_t)nstripes + 1), "allocating bounds");
  RQA_CUDA(cudaMemcpyAsync(ws->bounds, bounds, (nstripes + 1) * sizeof(int64_t),
                           cudaMemcpyHostToDevice, st),
           "copying bounds");
  UnitStitchArgs f;
  f.sp = d_prefix;
  f.ss = d_suffix;
  f.scol = reinterpret_cast<const uint2*>(d_col);
  f.srow = reinterpret_cast<const uint2*>(d_row);
  f.bounds = ws->bounds;
  f.nseg = nstripes;
  f.n = n;
  f.hist = hist;
  const int threads = 256;
  const int64_t blocks = std::min<int64_t>((n + threads - 1) / threads, 148 * 16);
  unit_fold_stripes<<<(int)blocks, threads, 0, st>>>(f);
  RQA_CUDA(cudaGetLastError(), "launching stitch kernel");
  g_launches++;
  return RQA_OK;
}

// Equal-area row stripes of the upper triangle, band aligned.
std::vector<int64_t> area_stripes(int64_t n, int g, int64_t band) {
  std::vector<int64_t> b(1, 0);
  for (int q = 1; q < g; ++q) {
    const double i = (double)n * (1.0 - std::sqrt(1.0 - (double)q / g));
    int64_t v = (int64_t)std::llround(i / band) * band;
    b.push_back(std::max(b.back(), std::min(n, v)));
  }
  b.push_back(n);
  return b;
}

// Full analysis on the current device; splits into sequential stripes (same
// code path as multi-GPU) when the summaries would not fit in memory.
int run_full(Workspace* ws, const Problem& p, unsigned long long* hist, unsigned long long* points,
             cudaStream_t st, cudaEvent_t ev_mid, char* err, size_t errlen) {
  size_t free_b = 0, total_b = 0;
  RQA_CUDA(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
  const double budget = 0.6 * (double)(free_b + ws->ps_cap * 2 + ws->cs_cap * 4);
  const double need = (double)unit_workspace_bytes(p, 0, p.n);
  int g = 1;
  while (need / g > budget && g < 64) g *= 2;
  if (g == 1)
    return launch_rows(ws, p, 0, p.n, kFoldFinal, hist, points, nullptr, nullptr, nullptr, nullptr,
                       st, ev_mid, err, errlen);
  const std::vector<int64_t> bounds = area_stripes(p.n, g, p.var.band_rows());
  const size_t per = (size_t)p.n;
  RQA_CUDA(grow(&ws->stripe_buf, &ws->stripe_buf_cap, (size_t)g * per * 4 + 2 * per),
           "allocating stripe summaries");
  int32_t* pre = ws->stripe_buf;
  int32_t* suf = pre + (size_t)g * per;
  uint32_t* col = reinterpret_cast<uint32_t*>(suf + (size_t)g * per);
  uint32_t* row = col + (size_t)g * 2 * per;
  RQA_CUDA(cudaMemsetAsync(row, 0, 2 * per * sizeof(uint32_t), st), "memset row parts");
  for (int q = 0; q < g; ++q) {
    const int rc = launch_rows(ws, p, bounds[q], bounds[q + 1], kFoldStripe, hist, points,
                               pre + (size_t)q * per, suf + (size_t)q * per,
                               col + (size_t)q * 2 * per, row, st, nullptr, err, errlen);
    if (rc) return rc;
  }
  if (ev_mid) RQA_CUDA(cudaEventRecord(ev_mid, st), "event");
  return stitch_stripes(ws, pre, suf, col, row, bounds.data(), g, p.n, hist, st, err, errlen);
}

// FP64 pipe microbenchmark: 8 independent DADD (or DMUL) chains per thread.
template <int OP>
__global__ void fp64_peak_kernel(double* out, int iters, double a) {
  double x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = OP == 0 ? __dadd_rn(x[j], a) : __dmul_rn(x[j], a);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

}  // namespace

void note_launch() { g_launches++; }

}  // namespace rqa

using namespace rqa;

extern "C" {

int rqa_version(void) { return 10000; }

int rqa_device_count(void) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return c;
}

int64_t rqa_launch_counter(void) { return g_launches.load(); }

int rqa_threshold(int32_t metric, int32_t m, double radius, double* thr) {
  if (!thr || metric < 0 || metric > 2 || m < 1 || !(radius >= 0)) return RQA_EINVAL;
  *thr = threshold_for(metric, m, radius);
  return RQA_OK;
}

int rqa_band_rows(int32_t metric, int32_t m, int32_t tau, int64_t n, int64_t* band_rows,
                  int32_t* reuse_kernel) {
  Variant v;
  if (m < 1 || tau < 1 || metric < 0 || metric > 2 || n < 1 ||
      !find_variant(metric, m, tau, n, &v))
    return RQA_EINVAL;
  if (band_rows) *band_rows = v.band_rows();
  if (reuse_kernel) *reuse_kernel = v.reuse;
  return RQA_OK;
}

int rqa_run(const double* series, int64_t len, int32_t m, int32_t tau, int32_t metric,
            double radius, int64_t theiler, int32_t device, int64_t* diag, int64_t* vert,
            int64_t* white, int64_t* points, double* timing, char* err, size_t errlen) {
  if (!series || !diag || !vert || !white || !points)
    return set_err(err, errlen, "null pointer argument"), RQA_EINVAL;
  Problem p;
  int rc = validate(len, m, tau, metric, radius, theiler, &p, err, errlen);
  if (rc) return rc;
  int ndev = rqa_device_count();
  if (ndev <= 0) return set_err(err, errlen, "no CUDA device available"), RQA_EDEVICE;
  if (device < 0 || device >= ndev)
    return set_err(err, errlen, "device %d out of range (%d visible)", device, ndev), RQA_EINVAL;
  RQA_CUDA(cudaSetDevice(device), "cudaSetDevice");
  Workspace* ws = workspace(device);
  std::lock_guard<std::mutex> lk(ws->mu);
  if (!ws->init) {
    RQA_CUDA(cudaStreamCreateWithFlags(&ws->stream, cudaStreamNonBlocking), "stream");
    for (auto& e : ws->ev) RQA_CUDA(cudaEventCreate(&e), "event");
    ws->init = true;
  }
  cudaStream_t st = ws->stream;
  const size_t hn = (size_t)(p.n + 1);
  RQA_CUDA(grow(&ws->hist, &ws->hist_cap, 3 * hn + 1), "allocating histograms");
  RQA_CUDA(cudaEventRecord(ws->ev[0], st), "event");
  rc = stage_series(ws, p, series, cudaMemcpyHostToDevice, st, err, errlen);
  if (rc) return rc;
  RQA_CUDA(cudaMemsetAsync(ws->hist, 0, (3 * hn + 1) * sizeof(unsigned long long), st), "memset");
  RQA_CUDA(cudaEventRecord(ws->ev[1], st), "event");
  rc = run_full(ws, p, ws->hist, ws->hist + 3 * hn, st, ws->ev[2], err, errlen);
  if (rc) return rc;
  RQA_CUDA(cudaEventRecord(ws->ev[3], st), "event");
  RQA_CUDA(cudaMemcpyAsync(diag, ws->hist, hn * 8, cudaMemcpyDeviceToHost, st), "d2h");
  RQA_CUDA(cudaMemcpyAsync(vert, ws->hist + hn, hn * 8, cudaMemcpyDeviceToHost, st), "d2h");
  RQA_CUDA(cudaMemcpyAsync(white, ws->hist + 2 * hn, hn * 8, cudaMemcpyDeviceToHost, st), "d2h");
  RQA_CUDA(cudaMemcpyAsync(points, ws->hist + 3 * hn, 8, cudaMemcpyDeviceToHost, st), "d2h");
  RQA_CUDA(cudaEventRecord(ws->ev[4], st), "event");
  RQA_CUDA(cudaStreamSynchronize(st), "running kernels");
  if (timing) {
    float ms[4] = {0, 0, 0, 0};
    cudaEventElapsedTime(&ms[0], ws->ev[0], ws->ev[1]);
    cudaEventElapsedTime(&ms[1], ws->ev[1], ws->ev[2]);
    cudaEventElapsedTime(&ms[2], ws->ev[2], ws->ev[3]);
    cudaEventElapsedTime(&ms[3], ws->ev[3], ws->ev[4]);
    float tot = 0;
    cudaEventElapsedTime(&tot, ws->ev[0], ws->ev[4]);
    for (int q = 0; q < 4; ++q) timing[q] = ms[q] * 1e-3;
    timing[4] = tot * 1e-3;
    const double kern = (ms[1] + ms[2]) * 1e-3;
    timing[5] = kern > 0 ? (double)p.n * (double)p.n / kern : 0.0;
    timing[6] = (double)p.var.band_rows();
    timing[7] = (double)((p.n + p.var.band_rows() - 1) / p.var.band_rows());
  }
  return RQA_OK;
}

int rqa_run_device(const double* d_series, int64_t len, int32_t m, int32_t tau, int32_t metric,
                   double radius, int64_t theiler, int64_t row_lo, int64_t row_hi, int32_t mode,
                   int64_t* d_hist, int64_t* d_points, int32_t* d_stripe_prefix,
                   int32_t* d_stripe_suffix, uint32_t* d_stripe_col, uint32_t* d_rowlead,
                   void* stream, char* err, size_t errlen) {
  if (!d_series || !d_hist || !d_points)
    return set_err(err, errlen, "null pointer argument"), RQA_EINVAL;
  Problem p;
  int rc = validate(len, m, tau, metric, radius, theiler, &p, err, errlen);
  if (rc) return rc;
  if (mode != kFoldFinal && mode != kFoldStripe)
    return set_err(err, errlen, "mode must be 0 (final) or 1 (stripe)"), RQA_EINVAL;
  if (row_lo < 0 || row_hi > p.n || row_lo > row_hi)
    return set_err(err, errlen, "row range [%lld, %lld) outside [0, %lld)", (long long)row_lo,
                   (long long)row_hi, (long long)p.n),
           RQA_EINVAL;
  if (mode == kFoldFinal && (row_lo != 0 || row_hi != p.n))
    return set_err(err, errlen, "final mode needs the full row range"), RQA_EINVAL;
  if (mode == kFoldStripe && (!d_stripe_prefix || !d_stripe_suffix || !d_stripe_col || !d_rowlead))
    return set_err(err, errlen, "stripe mode needs prefix/suffix/column/row-lead outputs"),
           RQA_EINVAL;
  int dev = 0;
  RQA_CUDA(cudaGetDevice(&dev), "cudaGetDevice");
  Workspace* ws = workspace(dev);
  std::lock_guard<std::mutex> lk(ws->mu);
  cudaStream_t st = (cudaStream_t)stream;
  rc = stage_series(ws, p, d_series, cudaMemcpyDeviceToDevice, st, err, errlen);
  if (rc) return rc;
  const size_t hn = (size_t)(p.n + 1);
  (void)hn;
  if (mode == kFoldFinal)
    return run_full(ws, p, reinterpret_cast<unsigned long long*>(d_hist),
                    reinterpret_cast<unsigned long long*>(d_points), st, nullptr, err, errlen);
  return launch_rows(ws, p, row_lo, row_hi, mode, reinterpret_cast<unsigned long long*>(d_hist),
                     reinterpret_cast<unsigned long long*>(d_points), d_stripe_prefix,
                     d_stripe_suffix, d_stripe_col, d_rowlead, st, nullptr, err, errlen);
}

int rqa_stitch_device(const int32_t* d_prefix, const int32_t* d_suffix, const uint32_t* d_col,
                      const uint32_t* d_rowpart, const int64_t* bounds, int32_t nstripes,
                      int64_t n, int64_t* d_hist, void* stream, char* err, size_t errlen) {
  if (!d_prefix || !d_suffix || !d_col || !d_rowpart || !bounds || !d_hist || nstripes < 1 || n < 1)
    return set_err(err, errlen, "invalid stitch arguments"), RQA_EINVAL;
  if (bounds[0] != 0 || bounds[nstripes] != n)
    return set_err(err, errlen, "stripes must cover rows [0, n)"), RQA_EINVAL;
  for (int g = 0; g < nstripes; ++g)
    if (bounds[g + 1] < bounds[g])
      return set_err(err, errlen, "stripe bounds must be non-decreasing"), RQA_EINVAL;
  int dev = 0;
  RQA_CUDA(cudaGetDevice(&dev), "cudaGetDevice");
  Workspace* ws = workspace(dev);
  std::lock_guard<std::mutex> lk(ws->mu);
  cudaStream_t st = (cudaStream_t)stream;
  const int rc = stitch_stripes(ws, d_prefix, d_suffix, d_col, d_rowpart, bounds, nstripes, n,
                                reinterpret_cast<unsigned long long*>(d_hist), st, err, errlen);
  if (rc) return rc;
  RQA_CUDA(cudaStreamSynchronize(st), "stitch");
  return RQA_OK;
}

int rqa_fp64_peak(int32_t device, double* dadd_per_s, double* dmul_per_s, char* err,
                  size_t errlen) {
  if (rqa_device_count() <= device || device < 0)
    return set_err(err, errlen, "no such CUDA device"), RQA_EDEVICE;
  RQA_CUDA(cudaSetDevice(device), "cudaSetDevice");
  int sms = 0;
  RQA_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device), "attr");
  double* out = nullptr;
  RQA_CUDA(cudaMalloc(&out, sizeof(double)), "malloc");
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  double res[2] = {0, 0};
  for (int op = 0; op < 2; ++op) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      if (op == 0) fp64_peak_kernel<0><<<blocks, threads>>>(out, iters, 1.0000001);
      else fp64_peak_kernel<1><<<blocks, threads>>>(out, iters, 1.0000001);
      cudaEventRecord(e1);
      RQA_CUDA(cudaEventSynchronize(e1), "fp64 peak kernel");
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double ops = (double)blocks * threads * iters * 8;
      res[op] = std::max(res[op], ops / (ms * 1e-3));
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (dadd_per_s) *dadd_per_s = res[0];
  if (dmul_per_s) *dmul_per_s = res[1];
  return RQA_OK;
}

int rqa_release(void) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  for (size_t d = 0; d < g_ws.size(); ++d) {
    Workspace* ws = g_ws[d];
    if (!ws) continue;
    cudaSetDevice((int)d);
    cudaFree(ws->s_pad);
    cudaFree(ws->ps);
    cudaFree(ws->cs);
    cudaFree(ws->rowlead);
    cudaFree(ws->rowpiece);
    cudaFree(ws->units);
    cudaFree(ws->units_bb);
    cudaFree(ws->band_start);
    cudaFree(ws->stripe_buf);
    cudaFree(ws->hist);
    cudaFree(ws->bounds);
    if (ws->init) {
      for (auto& e : ws->ev) cudaEventDestroy(e);
      cudaStreamDestroy(ws->stream);
    }
    delete ws;
    g_ws[d] = nullptr;
  }
  return RQA_OK;
}

}  // extern "C"
