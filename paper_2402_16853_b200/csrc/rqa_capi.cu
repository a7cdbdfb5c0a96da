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
  uint32_t* rowlead = nullptr; // [n]
  size_t rowlead_cap = 0;
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

// Upper-triangle band kernel over rows [row_lo, row_hi) + folds.
//   final mode: diagonal and hook folds write the complete histograms;
//   stripe mode: per-stripe summaries for rqa_stitch_device (multi-GPU).
int launch_rows(Workspace* ws, const Problem& p, int64_t row_lo, int64_t row_hi, int mode,
                unsigned long long* hist, unsigned long long* points, int32_t* out_p,
                int32_t* out_s, uint32_t* out_col, uint32_t* rowlead, cudaStream_t st,
                cudaEvent_t ev_mid, char* err, size_t errlen) {
  const int64_t H = p.var.band_rows();
  const int64_t nb = (row_hi - row_lo + H - 1) / H;
  if (nb <= 0) return RQA_OK;
  const int64_t total = sym_band_offset(nb, p.n, row_lo, H);  // compact entries
  RQA_CUDA(grow(&ws->ps, &ws->ps_cap, (size_t)(2 * total)), "allocating band summaries");
  RQA_CUDA(grow(&ws->cs, &ws->cs_cap, (size_t)total), "allocating column summaries");
  if (!rowlead) {
    RQA_CUDA(grow(&ws->rowlead, &ws->rowlead_cap, (size_t)p.n), "allocating row leads");
    rowlead = ws->rowlead;
  }
  SymArgs a;
  a.s = ws->s_pad + p.pad;
  a.len = p.len;
  a.n = p.n;
  a.row_lo = row_lo;
  a.row_hi = row_hi;
  a.thr = p.thr;
  a.theiler = p.theiler;
  a.m = p.m;
  a.tau = p.tau;
  a.P = ws->ps;
  a.S = ws->ps + total;
  a.colsum = ws->cs;
  a.rowlead = rowlead;
  a.hist = hist;
  a.points = points;
  static const char* skip_env = getenv("RQA_SKIP");  // profiling only: skip phases
  a.skip = skip_env ? atoi(skip_env) : 0;
  static const bool timers = getenv("RQA_TIMERS") != nullptr;  // profiling only: phase cycles
  a.timers = nullptr;
  if (timers) {
    RQA_CUDA(cudaMalloc(&a.timers, 4 * sizeof(unsigned long long)), "timers");
    RQA_CUDA(cudaMemsetAsync(a.timers, 0, 4 * sizeof(unsigned long long), st), "timers");
  }
  RQA_CUDA(p.var.launch(a, (int)nb, p.var.w, st), "launching band kernel");
  if (timers) {
    unsigned long long t[4];
    RQA_CUDA(cudaMemcpyAsync(t, a.timers, sizeof t, cudaMemcpyDeviceToHost, st), "timers");
    RQA_CUDA(cudaStreamSynchronize(st), "timers");
    const double tot = (double)(t[0] + t[1] + t[2] + t[3]);
    fprintf(stderr, "phase cycles (warp-summed): compute %.3f rows %.3f cols %.3f other %.3f\n",
            t[0] / tot, t[1] / tot, t[2] / tot, t[3] / tot);
    cudaFree(a.timers);
  }
  g_launches++;
  if (ev_mid) RQA_CUDA(cudaEventRecord(ev_mid, st), "event");

  SymFoldArgs f;
  memset(&f, 0, sizeof f);
  f.P = a.P;
  f.S = a.S;
  f.colsum = a.colsum;
  f.row_lo = row_lo;
  f.row_hi = row_hi;
  f.H = H;
  f.nb = (int)nb;
  f.rowlead = rowlead;
  f.n = p.n;
  f.hist = hist;
  f.out_p = out_p;
  f.out_s = out_s;
  f.out_col = reinterpret_cast<uint2*>(out_col);
  const int threads = 256;
  const int64_t blocks = std::min<int64_t>((p.n + threads - 1) / threads, 148 * 16);
  sym_fold_diag<<<(int)blocks, threads, 0, st>>>(f, mode);
  RQA_CUDA(cudaGetLastError(), "launching diagonal fold");
  sym_fold_hooks<<<(int)blocks, threads, 0, st>>>(f, mode);
  RQA_CUDA(cudaGetLastError(), "launching hook fold");
  g_launches += 2;
  return RQA_OK;
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
  rc = launch_rows(ws, p, 0, p.n, kFoldFinal, ws->hist, ws->hist + 3 * hn, nullptr, nullptr,
                   nullptr, nullptr, st, ws->ev[2], err, errlen);
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
  return launch_rows(ws, p, row_lo, row_hi, mode, reinterpret_cast<unsigned long long*>(d_hist),
                     reinterpret_cast<unsigned long long*>(d_points), d_stripe_prefix,
                     d_stripe_suffix, mode == kFoldStripe ? d_stripe_col : nullptr,
                     mode == kFoldStripe ? d_rowlead : nullptr, st, nullptr, err, errlen);
}

int rqa_stitch_device(const int32_t* d_prefix, const int32_t* d_suffix, const uint32_t* d_col,
                      const uint32_t* d_rowlead, const int64_t* bounds, int32_t nstripes, int64_t n,
                      int64_t* d_hist, void* stream, char* err, size_t errlen) {
  if (!d_prefix || !d_suffix || !d_col || !d_rowlead || !bounds || !d_hist || nstripes < 1 || n < 1)
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
  RQA_CUDA(grow(&ws->bounds, &ws->bounds_cap, (size_t)nstripes + 1), "allocating bounds");
  RQA_CUDA(cudaMemcpyAsync(ws->bounds, bounds, (nstripes + 1) * sizeof(int64_t),
                           cudaMemcpyHostToDevice, st),
           "copying bounds");
  SymFoldArgs f;
  memset(&f, 0, sizeof f);
  f.sp = d_prefix;
  f.ss = d_suffix;
  f.scol = reinterpret_cast<const uint2*>(d_col);
  f.bounds = ws->bounds;
  f.nseg = nstripes;
  f.rowlead = d_rowlead;
  f.n = n;
  f.hist = reinterpret_cast<unsigned long long*>(d_hist);
  const int threads = 256;
  const int64_t blocks = std::min<int64_t>((n + threads - 1) / threads, 148 * 16);
  sym_fold_stripes<<<(int)blocks, threads, 0, st>>>(f);
  RQA_CUDA(cudaGetLastError(), "launching stitch kernel");
  g_launches++;
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
