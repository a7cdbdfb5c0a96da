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
#include <chrono>
#include <mutex>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/rqa_b200.h"
#include "rqa_fold.cuh"
#include "rqa_variants.cuh"

namespace rqa {
namespace {

// Runtime knob: the variable's value, or nullptr when it is unset or empty
// (an empty RQA_WAVES= or RQA_PREFILTER= means "default", not 0).
const char* env_knob(const char* name) {
  const char* v = getenv(name);
  return (v && v[0]) ? v : nullptr;
}

// NVTX range over a host-side phase (header-only NVTX 3: free without a
// profiler attached; nsys / ncu --nvtx show the phases of every call).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

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

// Prefilter bound D*: acc <= T forces every term <= T, i.e. |d| <= D* with
// D* = max{x >= 0 : fl(x * x) <= T} for L2 (terms d*d), T for L1 (terms |d|).
double prefilter_bound(int metric, double T) {
  if (metric != kL2) return T;
  if (!(T >= 0) || std::isinf(T)) return T;
  // fl(x * x) is monotone in x >= 0, and so is the bit pattern of x: binary
  // search the largest pattern whose square rounds to <= T (T = 0 included,
  // where every x below ~2^-537 squares to 0)
  uint64_t lo = 0, hi = 0x7ff0000000000000ull;  // fl(0*0) <= T; inf*inf > T
  while (hi - lo > 1) {
    const uint64_t mid = lo + (hi - lo) / 2;
    double x;
    memcpy(&x, &mid, sizeof x);
    if (x * x <= T) lo = mid;
    else hi = mid;
  }
  double x;
  memcpy(&x, &lo, sizeof x);
  return x;
}

// fp32-mode threshold: T*32 = max{x : sqrtf(x) <= fl32(eps)} for L2 with
// m > 1, else fl32(radius) (numpy float32 semantics, oracle/rqa_oracle.c).
float threshold_for32(int metric, int m, double radius) {
  const float eps = (float)radius;
  if (!(metric == kL2 && m > 1)) return eps;
  if (std::isinf(eps)) return INFINITY;
  float t = eps * eps;
  if (std::isinf(t)) t = FLT_MAX;
  while (t > 0.0f && std::sqrt(t) > eps) t = std::nextafter(t, 0.0f);
  for (;;) {
    const float u = std::nextafter(t, INFINITY);
    if (std::isinf(u) || std::sqrt(u) > eps) break;
    t = u;
  }
  return t;
}

struct Workspace {
  std::mutex mu;
  cudaStream_t stream = nullptr;
  double* s_pad = nullptr;
  size_t s_cap = 0;  // elements
  float* sf_pad = nullptr;     // f32 filter: samples rounded to float32
  size_t sf_cap = 0;
  unsigned long long* maxbits = nullptr;  // [1]: prefilter sampling hit counter
  unsigned long long* stats = nullptr;    // [2]: max finite |s| (float64 bits), non-finite flag
  size_t stats_cap = 0;
  uint16_t* ps = nullptr;      // P and S (compact band layout)
  size_t ps_cap = 0;  // elements
  uint32_t* cs = nullptr;      // column-part summaries (compact band layout)
  size_t cs_cap = 0;
  uint32_t* rowlead = nullptr; // [2n] row part per row (single-device final mode)
  size_t rowlead_cap = 0;
  uint2* rowpiece = nullptr;   // [nunits][H]
  size_t rowpiece_cap = 0;
  uint2* drec = nullptr;       // [nunits][R-1][D] diagonal pieces cut at unit ends
  size_t drec_cap = 0;
  Unit* units = nullptr;       // [nunits] launch order
  size_t units_cap = 0;
  int4* units_bb = nullptr;    // [nunits] sorted by band, xa
  size_t units_bb_cap = 0;
  int32_t* band_start = nullptr;
  size_t band_start_cap = 0;
  int32_t* stripe_buf = nullptr;  // auto-striping: [G][n] x2 + [G][2n] + [2n]
  size_t stripe_buf_cap = 0;
  unsigned long long* hist = nullptr;
  size_t hist_cap = 0;  // elements (3*(n+1) + 2: points, fp32 mismatches)
  size_t maxbits_cap = 0;
  int64_t* bounds = nullptr;
  size_t bounds_cap = 0;
  int32_t* gather = nullptr;   // multi-device: gathered stripe summaries (device 0 only)
  size_t gather_cap = 0;
  unsigned long long* bins = nullptr;  // sparse D2H: [1 counter word][2 * kSparseCap pairs]
  size_t bins_cap = 0;
  cudaEvent_t ev[6] = {};
  bool init = false;
  unsigned long long* host_stats = nullptr;  // pinned [4]: f32 stats + sampled hits (one D2H)
  // last unit plan uploaded (reused while the geometry is unchanged: no
  // host planning or H2D copy inside repeated runs)
  int64_t plan_key[8] = {-1, -1, -1, -1, -1, -1, -1, -1};
  int64_t plan_nunits = 0;
};

// Resident CTAs per SM of a kernel variant (queried once per kernel and device).
int variant_occupancy(const Variant& v, int* per_sm) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<const void*, int>, int>> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const std::pair<const void*, int> key(v.kernel, dev);
  std::lock_guard<std::mutex> lk(mu);
  for (const auto& e : cache)
    if (e.first == key) return *per_sm = e.second, 0;
  cudaError_t e = cudaFuncSetAttribute(v.kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)v.smem);
  if (e == cudaSuccess)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, v.kernel, 32 * v.nw, v.smem);
  if (e != cudaSuccess) return (int)e;
  cache.emplace_back(key, *per_sm);
  return 0;
}

std::mutex g_ws_mu;
std::vector<Workspace*> g_ws;        // [slot * kMaxDevices + device]
constexpr int kMaxDevices = 64;      // per-process device ids
constexpr int kMaxSlots = 64;        // stripes of one multi-device call on the same device

// Workspace of (device, slot): slot > 0 only for the extra stripes a
// multi-device call places on a device it already uses.
Workspace* workspace(int dev, int slot = 0) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  const size_t key = (size_t)slot * kMaxDevices + (size_t)dev;
  if (g_ws.size() <= key) g_ws.resize(key + 1, nullptr);
  if (!g_ws[key]) g_ws[key] = new Workspace();
  return g_ws[key];
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
  // precision (rqa_unit.cuh f32 filter)
  int precision = 64;   // 64 or 32 (fp32 mode)
  int filt = -1;        // -1: float64 kernel; 0: f32 filter, exact; 1: fp32 mode
  float c32 = 0.f, band32 = 0.f, thr32 = 0.f;
  int all_amb = 0;
  const float* sf = nullptr;
  unsigned long long* mism = nullptr;
  double dstar = 0.0;   // prefilter bound (var.prec == 2)
  double cand = -1.0;   // sampled prefilter candidate fraction (-1: not sampled)
  float pre_negd2 = 0.f;  // -D2 of the packed float32 prefilter predicate
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
  if (p->n >= (int64_t)1 << 28)  // run lengths travel in 28 bits (rqa_runs.cuh events)
    return set_err(err, errlen, "n_vectors %lld exceeds 2^28 - 1", (long long)p->n), RQA_EINVAL;
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
  // padding for every geometry (f32 variants may use other band heights)
  const int64_t H = std::max<int64_t>(p->var.band_rows(), 1024), D = 256;
  p->pad = 2 * H + 4 * D + p->var.w + 256;
  return RQA_OK;
}

// Certified band of the f32 filter.  With M = max|s| (finite data) every
// float32 difference is bounded against its float64 counterpart (u = 2^-24,
// v = 2^-53, eta = 2^-149 absolute for float32 subnormals):
//   |d32 - d64| <= dd = 4.5 u M + 4 v M + 4 eta   (rounded inputs + subtraction)
// The float64 decision is acc64 <= T64, the float32 one acc32 - c32 < 0.
// Suppose |acc32 - c32| > B and the decisions differ.  Either acc32 < c32,
// or acc64 <= T64; in both cases every (non-negative) term of that sum is at
// most T'' = max(c32, T64) (1 + 4 m u), so |d| <= sqrt(T'') + dd for both
// precisions, and
//   L2:  |acc32 - acc64| <= E = m [dd (2 sqrt(T'') + dd) + (u + v) T''] + (m-1)(u + v) T'' 1.01
//   L1:  E = m dd + (m-1)(u + v) T'' 1.01
//   L-inf / m = 1 (per component): E = dd
// (+ 3 m eta for float32 underflow).  With B >= E + |c32 - T64| the first
// case gives acc64 < c32 - B + E <= T64 and the second acc32 <= T64 + E <
// c32 + B: both contradict.  B carries a further safety factor 2.  Cells
// whose float32 sum overflows are far outside the band and out in both
// precisions (T64 <= 1e30).
bool f32_band(const Problem& p, double maxabs, bool finite, float c32, float* band) {
  const double u = std::ldexp(1.0, -24), v = std::ldexp(1.0, -53), eta = std::ldexp(1.0, -149);
  const double M = maxabs, m = p.m;
  if (!finite || !(M <= 1e15) || !std::isfinite(c32) || !(c32 >= 1e-30f) || !(c32 <= 1e30f) ||
      !(p.thr <= 1e30))
    return false;
  const double dd = 4.5 * u * M + 4.0 * v * M + 4.0 * eta;
  const double T2 = std::max((double)c32, p.thr) * (1.0 + 4.0 * m * u);
  double E;
  if (p.metric == kL2 && p.m > 1) {
    E = m * (dd * (2.0 * std::sqrt(T2) + dd) + (u + v) * T2) + (m - 1.0) * (u + v) * T2 * 1.01;
  } else if (p.metric == kL1 && p.m > 1) {
    E = m * dd + (m - 1.0) * (u + v) * T2 * 1.01;
  } else {
    E = dd;
  }
  E += 3.0 * m * eta;
  const double B = 2.0 * (E + std::fabs((double)c32 - p.thr)) + eta;
  if (!(B < 1e30)) return false;
  *band = std::nextafter((float)B, INFINITY);
  return true;
}

// Fraction of prefilter candidates on pseudo-random cells (i, j): all m
// components within D*.  One thread per sample, counts into *hits.
__global__ void sample_candidates_kernel(const double* __restrict__ s, int64_t n, int m, int tau,
                                         double dstar, int samples, unsigned long long* hits) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= samples) return;
  uint64_t h = 0x9E3779B97F4A7C15ull * (uint64_t)(q + 1);
  h ^= h >> 31;
  h *= 0xBF58476D1CE4E5B9ull;
  h ^= h >> 29;
  const int64_t i = (int64_t)((h & 0xffffffffull) % (uint64_t)n);
  const int64_t j = (int64_t)((h >> 32) % (uint64_t)n);
  bool c = true;
  for (int k = 0; k < m && c; ++k)
    c = fabs(__dsub_rn(s[i + (int64_t)k * tau], s[j + (int64_t)k * tau])) <= dstar;
  if (c) atomicAdd(hits, 1ull);
}

// Nonzero histogram bins as (index, count) pairs (sparse D2H of the results).
__global__ void compact_bins_kernel(const unsigned long long* __restrict__ h, int64_t count,
                                    unsigned long long* __restrict__ out, unsigned int* counter,
                                    unsigned int cap) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < count;
       q += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long v = h[q];
    if (v) {
      const unsigned int slot = atomicAdd(counter, 1u);
      if (slot < cap) {
        out[2 * (size_t)slot] = (unsigned long long)q;
        out[2 * (size_t)slot + 1] = v;
      }
    }
  }
}

// dst += src over count counters (multi-device histogram reduction on the
// first device; src is a peer copy or another stripe's workspace there).
__global__ void hist_accumulate_kernel(unsigned long long* __restrict__ dst,
                                       const unsigned long long* __restrict__ src, int64_t count) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < count;
       q += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long v = src[q];
    if (v) dst[q] += v;
  }
}

// float32 copy of the series; out[0] = max |s| over the finite samples (as
// float64 bits), out[1] = 1 if any sample is NaN or infinite.
__global__ void prep_f32_kernel(const double* __restrict__ s, float* __restrict__ sf, int64_t count,
                                unsigned long long* out) {
  unsigned long long mx = 0;
  bool nonfinite = false;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < count;
       q += (int64_t)gridDim.x * blockDim.x) {
    const double x = s[q];
    sf[q] = __double2float_rn(x);
    const unsigned long long b = (unsigned long long)__double_as_longlong(x) & 0x7fffffffffffffffull;
    if (b >= 0x7ff0000000000000ull) nonfinite = true;
    else mx = b > mx ? b : mx;
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const unsigned long long y = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = y > mx ? y : mx;
  }
  nonfinite = __any_sync(0xffffffffu, nonfinite);
  if ((threadIdx.x & 31) == 0) {
    if (mx) atomicMax(out, mx);
    if (nonfinite) atomicOr(out + 1, 1ull);
  }
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
  NvtxRange nvtx_("rqa.stage_series");
  const size_t need = (size_t)(p.len + 2 * p.pad);
  RQA_CUDA(grow(&ws->s_pad, &ws->s_cap, need), "allocating series buffer");
  RQA_CUDA(cudaMemsetAsync(ws->s_pad, 0, (size_t)p.pad * sizeof(double), st), "memset pad");
  RQA_CUDA(cudaMemsetAsync(ws->s_pad + p.pad + p.len, 0, (size_t)p.pad * sizeof(double), st),
           "memset pad");
  RQA_CUDA(cudaMemcpyAsync(ws->s_pad + p.pad, src, (size_t)p.len * sizeof(double), kind, st),
           "copying series");
  return RQA_OK;
}

// float32 copy of the staged series (same padding) plus max |s| and whether
// every sample is finite; sets p->sf.  One small kernel + a 8-byte readback.
int stage_f32(Workspace* ws, Problem* p, cudaStream_t st, double* maxabs, bool* finite, char* err,
              size_t errlen) {
  const size_t count = (size_t)(p->len + 2 * p->pad);
  RQA_CUDA(grow(&ws->sf_pad, &ws->sf_cap, count), "allocating float32 series");
  RQA_CUDA(grow(&ws->stats, &ws->stats_cap, 2), "allocating");
  RQA_CUDA(cudaMemsetAsync(ws->stats, 0, 2 * sizeof(unsigned long long), st), "memset");
  prep_f32_kernel<<<148 * 4, 256, 0, st>>>(ws->s_pad, ws->sf_pad, (int64_t)count, ws->stats);
  RQA_CUDA(cudaGetLastError(), "launching f32 staging");
  g_launches++;
  unsigned long long mb[2] = {0, 0};
  RQA_CUDA(cudaMemcpyAsync(mb, ws->stats, sizeof mb, cudaMemcpyDeviceToHost, st), "d2h");
  RQA_CUDA(cudaStreamSynchronize(st), "f32 staging");
  *finite = mb[1] == 0;
  memcpy(maxabs, &mb[0], sizeof *maxabs);
  p->sf = ws->sf_pad + p->pad;
  return RQA_OK;
}

// Bound of the packed float32 prefilter predicate (kF32Pred kernels): with
// u = 2^-24 and M = max |s|, |d64| <= D* implies
//   |fl32(fl32(r) - fl32(c))| <= B = D* (1 + 2^-50) + u (2M + D*) (1 + 2^-20),
// so every component candidate of the float64 prefilter has d32^2 < D2 for
// the float D2 > B^2 returned here (fma(d32, d32, -D2) is then negative, its
// sign bit set).  NaN / infinite samples need no bound: every cell with such
// a component is non-recurrent in the reference (NaN or infinite sum), and
// whatever the float32 predicate says about it, the exact float64 sum of a
// candidate decides.  Returns false when the finite samples or the bound are
// out of range (|s| >= 1e30 would overflow float32): no prefilter then.
bool prefilter_f32_bound(double dstar, double maxabs, float* d2) {
  if (!(maxabs < 1e30) || !(dstar >= 0) || !(dstar < 1e18)) return false;
  const double u = std::ldexp(1.0, -24);
  const double B = dstar * (1.0 + std::ldexp(1.0, -50)) +
                   u * (2.0 * maxabs + dstar) * (1.0 + std::ldexp(1.0, -20)) +
                   4.0 * u * u * maxabs;
  const double B2 = B * B * (1.0 + std::ldexp(1.0, -40));
  if (!(B2 < 1e37)) return false;
  float f = (float)B2;
  if ((double)f < B2) f = std::nextafter(f, INFINITY);
  *d2 = std::nextafter(f, INFINITY);  // strictly above B^2
  return true;
}

// Precision plan after the series is staged: precision 32 always runs the f32
// kernels (fp32 mode).  Precision 64 runs the float64 kernels by default: the
// f32 filter issues 8 % fewer instructions on C3 but moves the evaluation
// from the otherwise idle FP64 pipe onto the FMA/ALU pipes the run
// bookkeeping saturates, and measured 3 % slower (profiles/r01_ncu_f32_vs_fp64.txt).
// RQA_FILTER=1 enables it when the band is certifiable and narrow (band <=
// 1e-2 of the threshold) and a packed variant exists; RQA_FILTER=2 drops the
// width condition (tests).  Results are bit-identical on every path.
int plan_precision(Workspace* ws, Problem* p, cudaStream_t st, char* err, size_t errlen) {
  p->filt = -1;
  static const char* fenv = env_knob("RQA_FILTER");
  const int want = fenv ? atoi(fenv) : 0;
  Variant fv;
  const bool packed = find_variant_f32(p->metric, p->m, p->tau, true, &fv);
  if (p->precision == 64 && (want == 0 || !packed)) return RQA_OK;
  double maxabs = 0.0;
  bool finite = false;
  int rc = stage_f32(ws, p, st, &maxabs, &finite, err, errlen);
  if (rc) return rc;
  if (p->precision == 32) {
    const float t32 = threshold_for32(p->metric, p->m, p->radius);
    p->thr32 = t32;
    p->c32 = std::nextafter(t32, INFINITY);
    p->all_amb = f32_band(*p, maxabs, finite, p->c32, &p->band32) ? 0 : 1;
    p->filt = 1;
    if (!find_variant_f32(p->metric, p->m, p->tau, false, &p->var))
      return set_err(err, errlen, "no fp32 kernel for this embedding"), RQA_EINVAL;
    return RQA_OK;
  }
  const float c = (float)p->thr;
  float band = 0.f;
  if (!f32_band(*p, maxabs, finite, c, &band)) return RQA_OK;
  if (want != 2 && !(band <= 1e-2f * c)) return RQA_OK;
  p->c32 = c;
  p->thr32 = std::nextafter(c, -INFINITY);  // acc32 <= thr32  <=>  acc32 < c32
  p->band32 = band;
  p->all_amb = 0;
  p->filt = 0;
  p->var = fv;
  return RQA_OK;
}

// Sparse prefilter plan (precision 64, float64 kernels): sample the fraction
// of cells whose m components all lie within D*; below prefilter_max(m) the
// prefilter kernel (AND of predicates + exact sums of the candidates) issues
// fewer instructions than the term-window kernel.  RQA_PREFILTER=0 disables,
// =1 forces it whenever a variant exists.  Results are identical either way.
// The exact term-reuse kernel costs about m + 2 FP64 ops per cell, the
// prefilter 2 plus the candidates' full sums, so its break-even candidate
// fraction grows with m.
inline double prefilter_max(int m) { return 0.05 * std::max(1.0, m / 3.0); }

int plan_prefilter(Workspace* ws, Problem* p, cudaStream_t st, char* err, size_t errlen) {
  NvtxRange nvtx_("rqa.plan_prefilter");
  if (p->precision != 64 || p->filt != -1) return RQA_OK;
  static const char* penv = env_knob("RQA_PREFILTER");
  const int want = penv ? atoi(penv) : 2;
  if (want == 0) return RQA_OK;
  Variant pv;
  if (!find_variant_pre(p->metric, p->m, p->tau, &pv)) return RQA_OK;
  // small matrices: the sampling round trip would cost more than it can save
  if (want != 1 && p->n < ((int64_t)1 << 15)) return RQA_OK;
  const double dstar = prefilter_bound(p->metric, p->thr);
  if (!(dstar >= 0) || std::isinf(dstar)) return RQA_OK;
  // one device round trip: the sampled candidate fraction (decides the
  // kernel) and, for the packed float32 predicate, max |s| of the staged
  // float32 series (bounds the predicate)
  const bool sample = want != 1;
  const int samples = 1 << 16;
  RQA_CUDA(grow(&ws->stats, &ws->stats_cap, 3), "allocating");
  if (!ws->host_stats)
    RQA_CUDA(cudaMallocHost(&ws->host_stats, 4 * sizeof(unsigned long long)), "allocating");
  RQA_CUDA(cudaMemsetAsync(ws->stats, 0, 3 * sizeof(unsigned long long), st), "memset");
  if (pv.f32pred) {
    const size_t count = (size_t)(p->len + 2 * p->pad);
    RQA_CUDA(grow(&ws->sf_pad, &ws->sf_cap, count), "allocating float32 series");
    prep_f32_kernel<<<148 * 4, 256, 0, st>>>(ws->s_pad, ws->sf_pad, (int64_t)count, ws->stats);
    RQA_CUDA(cudaGetLastError(), "launching f32 staging");
    g_launches++;
    p->sf = ws->sf_pad + p->pad;
  }
  if (sample) {
    sample_candidates_kernel<<<samples / 256, 256, 0, st>>>(ws->s_pad + p->pad, p->n, p->m,
                                                           p->tau, dstar, samples,
                                                           ws->stats + 2);
    RQA_CUDA(cudaGetLastError(), "launching candidate sampling");
    g_launches++;
  }
  if (sample || pv.f32pred) {
    RQA_CUDA(cudaMemcpyAsync(ws->host_stats, ws->stats, 3 * sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, st),
             "d2h");
    RQA_CUDA(cudaStreamSynchronize(st), "prefilter planning");
  }
  if (sample) {
    p->cand = (double)ws->host_stats[2] / samples;
    if (p->cand > prefilter_max(p->m)) return RQA_OK;
  }
  if (pv.f32pred) {
    double maxabs = 0.0;
    memcpy(&maxabs, &ws->host_stats[0], sizeof maxabs);
    float d2 = 0.f;
    if (!prefilter_f32_bound(dstar, maxabs, &d2)) return RQA_OK;
    p->pre_negd2 = -d2;
  }
  p->dstar = dstar;
  p->var = pv;
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
  // waves of units: more waves shorten the tail of the launch, fewer waves
  // recompute fewer boundary iterations (one per unit).  Measured optimum
  // (round 2): 32 waves for a whole 2^20 run (~7,100 iterations per resident
  // CTA), 16 for one of 8 stripes of it (~890): waves = 16 (T / 887)^(1/3),
  // T = iterations per resident CTA, clamped to [8, 64]; RQA_WAVES overrides
  static const char* wenv = env_knob("RQA_WAVES");
  const double per_slot = (double)total / std::max(1, slots);
  const int64_t waves = wenv ? std::max(1, atoi(wenv))
                             : std::min<int64_t>(64, std::max<int64_t>(
                                   8, std::llround(16.0 * std::cbrt(per_slot / 887.0))));
  // units of >= 16 iterations keep the recomputed iteration <= 1/16 of the
  // work, unless the whole triangle is too small to fill the GPU once (C1):
  // then parallelism wins over the recomputation
  static const char* menv = env_knob("RQA_MIN_UNIT");
  const int64_t min_len = menv ? std::max(1, atoi(menv))
                               : std::min<int64_t>(16, std::max<int64_t>(1, total / slots));
  int64_t len = std::max<int64_t>(min_len, total / std::max<int64_t>(1, waves * slots));
  // tail fraction (RQA_TAIL_FRAC, default 0.15): the last tf of every band's
  // sweep is cut into units of len/2 and the rest into units of 2 len, so the
  // longest-first launch order ends with small units (shorter tail) while
  // the unit count (boundary recomputation) stays about the same.  Sweep
  // 0 / 0.25 / 0.35 / 0.5: 0.25 best (C3 -0.3 %, P -0.7 %, C4 -1.1 %, one of 8
  // C3 stripes -1 % against 0); then 0.15 / 0.2 / 0.25 with the range-tested
  // kernels: 0.15 (C3 -0.12 %, C4 -0.24 %, C5 -0.05 %, P and stripes equal)
  static const char* tenv = env_knob("RQA_TAIL_FRAC");
  const double tf = tenv ? std::min(0.9, std::max(0.0, atof(tenv))) : 0.15;
  UnitPlan pl;
  pl.band_start.assign(nb + 1, 0);
  auto cut = [&](int64_t b, int64_t lo, int64_t hi, int64_t piece) {
    // every unit spans >= R iterations: a diagonal's band segment (R
    // consecutive iterations) is then cut by at most one unit boundary
    const int64_t w = hi - lo;
    const int64_t parts = std::max<int64_t>(1, std::min((w + piece - 1) / piece, w / R));
    for (int64_t q = 0; q < parts; ++q) {
      const int32_t xa = (int32_t)(lo + w * q / parts), xb = (int32_t)(lo + w * (q + 1) / parts);
      const int32_t idx = (int32_t)pl.units.size();
      pl.units.push_back(Unit{(int32_t)b, xa, xb, idx});
      pl.by_band.push_back(make_int4((int)b, xa, xb, idx));
    }
  };
  for (int64_t b = 0; b < nb; ++b) {
    pl.band_start[b] = (int32_t)pl.by_band.size();
    const int64_t split = X[b] - std::llround(X[b] * tf);
    if (tf > 0.0 && split >= R && X[b] - split >= R) {
      cut(b, 0, split, 2 * len);
      cut(b, split, X[b], std::max<int64_t>(R, len / 2));
    } else {
      cut(b, 0, X[b], len);
    }
  }
  pl.band_start[nb] = (int32_t)pl.by_band.size();
  std::stable_sort(pl.units.begin(), pl.units.end(),
                   [](const Unit& u, const Unit& v) { return (u.xb - u.xa) > (v.xb - v.xa); });
  return pl;
}

// Band-level summaries: P and S (uint16) and the column part (uint32) per
// (band, diagonal / column): 8 bytes per entry of the compact layout.
int64_t unit_workspace_bytes(const Problem& p, int64_t row_lo, int64_t row_hi) {
  const int64_t H = p.var.band_rows();
  const int64_t nb = (row_hi - row_lo + H - 1) / H;
  return sym_band_offset(nb, p.n, row_lo, H) * 8;
}

// Work-unit kernel over rows [row_lo, row_hi) + folds.
//   final mode: diagonal and hook folds write the complete histograms;
//   stripe mode: per-stripe summaries for the cross-stripe stitch.
int launch_rows(Workspace* ws, const Problem& p, int64_t row_lo, int64_t row_hi, int mode,
                unsigned long long* hist, unsigned long long* points, int32_t* out_p,
                int32_t* out_s, uint32_t* out_col, uint32_t* out_row, cudaStream_t st,
                cudaEvent_t ev_mid, char* err, size_t errlen) {
  NvtxRange nvtx_("rqa.launch_rows");
  const int64_t H = p.var.band_rows(), HS = p.var.slot_rows();
  const int64_t nb = (row_hi - row_lo + H - 1) / H;
  if (nb <= 0) return RQA_OK;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (int e = variant_occupancy(p.var, &per_sm)) return cuda_fail((cudaError_t)e, "occupancy", err, errlen);
  const int slots = sms * std::max(1, per_sm);
  const int64_t D = p.var.slot_rows(), R = p.var.r;
  const int64_t key[8] = {p.n, row_lo, row_hi, H, D, R, slots, (int64_t)p.var.nw};
  int64_t nunits = ws->plan_nunits;
  if (!std::equal(key, key + 8, ws->plan_key)) {
    // a new geometry: plan, upload (ordered on st before the kernel), remember
    const UnitPlan pl = plan_units(p, row_lo, row_hi, slots);
    nunits = (int64_t)pl.units.size();
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
    RQA_CUDA(cudaStreamSynchronize(st), "copying units");  // pageable sources go out of scope
    std::copy(key, key + 8, ws->plan_key);
    ws->plan_nunits = nunits;
  }
  const int64_t ctot = sym_band_offset(nb, p.n, row_lo, H);
  RQA_CUDA(grow(&ws->ps, &ws->ps_cap, (size_t)(2 * ctot)), "allocating diagonal summaries");
  RQA_CUDA(grow(&ws->drec, &ws->drec_cap, (size_t)(nunits * std::max<int64_t>(R - 1, 1) * D)),
           "allocating diagonal records");
  RQA_CUDA(grow(&ws->cs, &ws->cs_cap, (size_t)ctot), "allocating column summaries");
  RQA_CUDA(grow(&ws->rowpiece, &ws->rowpiece_cap, (size_t)(nunits * H)), "allocating row pieces");
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
  a.P = ws->ps;               // [2][ctot]: P then S, band-level compact layout
  a.S = ws->ps + ctot;
  a.colsum = ws->cs;
  a.rowlead = nullptr;
  a.hist = hist;
  a.points = points;
  static const char* skip_env = env_knob("RQA_SKIP");  // profiling only: skip phases
  a.skip = skip_env ? atoi(skip_env) : 0;
  static const char* flush_env = env_knob("RQA_FLUSH_EVERY");  // tests: power of two
  const int flush_every = flush_env ? std::max(1, atoi(flush_env)) : 4096;
  a.flush_mask = ((flush_every & (flush_every - 1)) == 0 ? flush_every : 4096) - 1;
  a.timers = nullptr;
  a.sf = p.sf;
  a.c32 = p.c32;
  a.band32 = p.band32;
  a.thr32 = p.thr32;
  a.prec_mode = p.filt == 1 ? 1 : 0;
  a.all_amb = p.all_amb;
  a.mism = p.mism;
  a.dstar = p.dstar;
  a.pre_negd2 = p.pre_negd2;
  ua.units = ws->units;
  ua.rowpiece = ws->rowpiece;
  ua.drec = ws->drec;
  ua.cap_ps = ctot;
  ua.cap_cs = ctot;
  ua.cap_drec = nunits * std::max<int64_t>(R - 1, 1) * D;
  ua.cap_piece = nunits * H;
  RQA_CUDA(p.var.launch(ua, (int)nunits, p.var.w, st), "launching band kernel");
  g_launches++;
  if (ev_mid) RQA_CUDA(cudaEventRecord(ev_mid, st), "event");

  const int threads = 256;
  if (R > 1 && nunits > nb) {  // some band is cut into several units
    DiagPieceArgs dp;
    dp.units_by_band = ws->units_bb;
    dp.nunits = (int)nunits;
    dp.drec = ws->drec;
    dp.P = a.P;
    dp.S = a.S;
    dp.row_lo = row_lo;
    dp.row_hi = row_hi;
    dp.n = p.n;
    dp.H = H;
    dp.HS = HS;
    dp.D = D;
    dp.R = (int)R;
    dp.hist = hist;
    dp.cap_ps = ctot;
    dp.cap_drec = nunits * (R - 1) * D;
    const int64_t recs = nunits * (R - 1) * D;
    fix_diag_pieces<<<(int)std::min<int64_t>((recs + threads - 1) / threads, 148 * 16), threads, 0,
                      st>>>(dp);
    RQA_CUDA(cudaGetLastError(), "launching diagonal piece join");
    g_launches++;
  }
  // fold threads take diagonals / hooks t and n-1-t
  const int64_t blocks = std::min<int64_t>(((p.n + 1) / 2 + threads - 1) / threads, 148 * 16);
  SymFoldArgs f;
  memset(&f, 0, sizeof f);
  f.P = a.P;
  f.S = a.S;
  f.row_lo = row_lo;
  f.row_hi = row_hi;
  f.H = H;                    // diagonal segments are bands
  f.nb = (int)nb;
  f.n = p.n;
  f.hist = hist;
  f.out_p = out_p;
  f.out_s = out_s;

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
  // one launch: the diagonal fold (about a fifth of the fold time) and the
  // hook fold share the grid
  static const char* dfrac = env_knob("RQA_FOLD_DIAG_SHARE");
  const double share = dfrac ? atof(dfrac) : 0.3;
  const int dblocks = (int)std::max<int64_t>(1, (int64_t)(blocks * share));
  unit_fold_all<<<(int)blocks + dblocks, threads, 0, st>>>(f, h, mode, dblocks);
  RQA_CUDA(cudaGetLastError(), "launching folds");
  g_launches += 1;
  return RQA_OK;
}

int stitch_stripes(Workspace* ws, const int32_t* d_prefix, const int32_t* d_suffix,
                   const uint32_t* d_col, const uint32_t* d_row, const int64_t* bounds,
                   int32_t nstripes, int64_t n, unsigned long long* hist, cudaStream_t st,
                   char* err, size_t errlen) {
  NvtxRange nvtx_("rqa.stitch");
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
  const double need = (double)unit_workspace_bytes(p, 0, p.n);
  int g = 1;
  if (need > (double)(ws->ps_cap * 2 + ws->cs_cap * 4)) {  // buffers must grow: check memory
    size_t free_b = 0, total_b = 0;
    RQA_CUDA(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
    const double budget = 0.6 * (double)(free_b + ws->ps_cap * 2 + ws->cs_cap * 4);
    while (need / g > budget && g < 64) g *= 2;
  }
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

// Results back to the caller: hist = [3][hn] histograms + points + mismatches
// on the current device.  With RQA_FLAG_OUT_ZEROED (caller's arrays are
// zero-filled) only the nonzero bins travel, compacted on the device; else
// dense copies.  Synchronous on st.
int copy_out(Workspace* ws, const unsigned long long* hist, size_t hn, int32_t flags, int64_t* diag,
             int64_t* vert, int64_t* white, int64_t* points, int64_t* mismatches, cudaStream_t st,
             char* err, size_t errlen) {
  NvtxRange nvtx_("rqa.copy_out");
  // outputs: the nonzero bins only when the caller's arrays are zero-filled
  // (RQA_FLAG_OUT_ZEROED) and they fit the pair buffer, else dense copies
  bool dense = true;
  if (flags & RQA_FLAG_OUT_ZEROED) {
    constexpr unsigned int kSparseCap = 1u << 20;
    RQA_CUDA(grow(&ws->bins, &ws->bins_cap, 1 + 2 * (size_t)kSparseCap), "allocating bins");
    unsigned int* counter = reinterpret_cast<unsigned int*>(ws->bins);
    RQA_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned long long), st), "memset");
    const int64_t nb3 = 3 * (int64_t)hn;
    compact_bins_kernel<<<(int)std::min<int64_t>((nb3 + 255) / 256, 148 * 8), 256, 0, st>>>(
        hist, nb3, ws->bins + 1, counter, kSparseCap);
    RQA_CUDA(cudaGetLastError(), "launching bin compaction");
    g_launches++;
    unsigned long long cnt = 0;
    RQA_CUDA(cudaMemcpyAsync(&cnt, ws->bins, sizeof cnt, cudaMemcpyDeviceToHost, st), "d2h");
    RQA_CUDA(cudaStreamSynchronize(st), "bin compaction");
    cnt &= 0xffffffffull;
    if (cnt <= kSparseCap) {
      std::vector<unsigned long long> pairs(2 * cnt + 2);
      if (cnt)
        RQA_CUDA(cudaMemcpyAsync(pairs.data(), ws->bins + 1, 2 * cnt * 8, cudaMemcpyDeviceToHost,
                                 st),
                 "d2h");
      RQA_CUDA(cudaStreamSynchronize(st), "d2h");
      int64_t* outs[3] = {diag, vert, white};
      for (unsigned long long q = 0; q < cnt; ++q) {
        const uint64_t idx = pairs[2 * q];
        outs[idx / hn][idx % hn] = (int64_t)pairs[2 * q + 1];
      }
      dense = false;
    }
  }
  if (dense) {
    RQA_CUDA(cudaMemcpyAsync(diag, hist, hn * 8, cudaMemcpyDeviceToHost, st), "d2h");
    RQA_CUDA(cudaMemcpyAsync(vert, hist + hn, hn * 8, cudaMemcpyDeviceToHost, st), "d2h");
    RQA_CUDA(cudaMemcpyAsync(white, hist + 2 * hn, hn * 8, cudaMemcpyDeviceToHost, st),
             "d2h");
  }
  RQA_CUDA(cudaMemcpyAsync(points, hist + 3 * hn, 8, cudaMemcpyDeviceToHost, st), "d2h");
  if (mismatches)
    RQA_CUDA(cudaMemcpyAsync(mismatches, hist + 3 * hn + 1, 8, cudaMemcpyDeviceToHost, st),
             "d2h");
  RQA_CUDA(cudaStreamSynchronize(st), "copying results");
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

// One stripe of a multi-device call, run by its own host thread.
struct StripeJob {
  int dev = 0, slot = 0;
  int64_t lo = 0, hi = 0;
  Workspace* ws = nullptr;
  unsigned long long* hist = nullptr;  // [3(n+1) + 2]: histograms, points, mismatches
  int32_t *pre = nullptr, *suf = nullptr;
  uint32_t *col = nullptr, *row = nullptr;
  float ms = 0.f;
  int rc = 0;
  char err[256] = {0};
  // evaluation path the stripe's plan chose (timing[6], [8..10])
  Variant var{};
  int filt = -1;
  float band32 = 0.f;
  double cand = -1.0;
};

int run_stripe_job(StripeJob* j, const Problem& p0, const double* series) {
  NvtxRange nvtx_("rqa.stripe_job");
  char* err = j->err;
  const size_t errlen = sizeof j->err;
  RQA_CUDA(cudaSetDevice(j->dev), "cudaSetDevice");
  Workspace* ws = j->ws;
  if (!ws->init) {
    RQA_CUDA(cudaStreamCreateWithFlags(&ws->stream, cudaStreamNonBlocking), "stream");
    for (auto& e : ws->ev) RQA_CUDA(cudaEventCreate(&e), "event");
    ws->init = true;
  }
  cudaStream_t st = ws->stream;
  Problem p = p0;
  const size_t hn = (size_t)(p.n + 1), n = (size_t)p.n;
  RQA_CUDA(grow(&ws->hist, &ws->hist_cap, 3 * hn + 2), "allocating histograms");
  RQA_CUDA(grow(&ws->stripe_buf, &ws->stripe_buf_cap, 6 * n), "allocating stripe summaries");
  j->hist = ws->hist;
  j->pre = ws->stripe_buf;
  j->suf = j->pre + n;
  j->col = reinterpret_cast<uint32_t*>(j->suf + n);
  j->row = j->col + 2 * n;
  int rc = stage_series(ws, p, series, cudaMemcpyHostToDevice, st, err, errlen);
  if (rc) return rc;
  RQA_CUDA(cudaMemsetAsync(ws->hist, 0, (3 * hn + 2) * sizeof(unsigned long long), st), "memset");
  RQA_CUDA(cudaMemsetAsync(j->row, 0, 2 * n * sizeof(uint32_t), st), "memset");
  rc = plan_precision(ws, &p, st, err, errlen);
  if (!rc) rc = plan_prefilter(ws, &p, st, err, errlen);
  if (rc) return rc;
  p.mism = ws->hist + 3 * hn + 1;
  RQA_CUDA(cudaEventRecord(ws->ev[1], st), "event");
  rc = launch_rows(ws, p, j->lo, j->hi, kFoldStripe, ws->hist, ws->hist + 3 * hn, j->pre, j->suf,
                   j->col, j->row, st, nullptr, err, errlen);
  if (rc) return rc;
  RQA_CUDA(cudaEventRecord(ws->ev[2], st), "event");
  RQA_CUDA(cudaStreamSynchronize(st), "stripe kernels");
  j->var = p.var;
  j->filt = p.filt;
  j->band32 = p.band32;
  j->cand = p.cand;
  cudaEventElapsedTime(&j->ms, ws->ev[1], ws->ev[2]);
  return RQA_OK;
}

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

int rqa_plan_units(int64_t n, int64_t row_lo, int64_t row_hi, int32_t slot_rows, int32_t r,
                   int32_t slots, int32_t* units, int64_t cap, int64_t* count) {
  if (!count || n < 1 || row_lo < 0 || row_hi > n || row_lo >= row_hi || slot_rows < 32 ||
      slot_rows % 32 != 0 || r < 1 || slots < 1 || (cap > 0 && !units))
    return RQA_EINVAL;
  Problem p;
  memset(&p.var, 0, sizeof p.var);
  p.n = n;
  p.var.nw = slot_rows / 32;
  p.var.r = r;
  const UnitPlan pl = plan_units(p, row_lo, row_hi, slots);
  *count = (int64_t)pl.by_band.size();
  for (int64_t q = 0; q < std::min<int64_t>(cap, *count); ++q) {
    units[3 * q] = pl.by_band[q].x;
    units[3 * q + 1] = pl.by_band[q].y;
    units[3 * q + 2] = pl.by_band[q].z;
  }
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

int rqa_run_prec(const double* series, int64_t len, int32_t m, int32_t tau, int32_t metric,
                 double radius, int64_t theiler, int32_t precision, int32_t device,
                 int32_t flags, int64_t* diag, int64_t* vert, int64_t* white, int64_t* points,
                 int64_t* mismatches, double* timing, char* err, size_t errlen) {
  NvtxRange nvtx_("rqa_run_prec");
  if (!series || !diag || !vert || !white || !points)
    return set_err(err, errlen, "null pointer argument"), RQA_EINVAL;
  if (precision != 64 && precision != 32)
    return set_err(err, errlen, "precision must be 64 or 32"), RQA_EINVAL;
  Problem p;
  int rc = validate(len, m, tau, metric, radius, theiler, &p, err, errlen);
  if (rc) return rc;
  p.precision = precision;
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
  RQA_CUDA(grow(&ws->hist, &ws->hist_cap, 3 * hn + 2), "allocating histograms");
  RQA_CUDA(cudaEventRecord(ws->ev[0], st), "event");
  rc = stage_series(ws, p, series, cudaMemcpyHostToDevice, st, err, errlen);
  if (rc) return rc;
  RQA_CUDA(cudaMemsetAsync(ws->hist, 0, (3 * hn + 2) * sizeof(unsigned long long), st), "memset");
  rc = plan_precision(ws, &p, st, err, errlen);
  if (!rc) rc = plan_prefilter(ws, &p, st, err, errlen);
  if (rc) return rc;
  p.mism = ws->hist + 3 * hn + 1;
  RQA_CUDA(cudaEventRecord(ws->ev[1], st), "event");
  rc = run_full(ws, p, ws->hist, ws->hist + 3 * hn, st, ws->ev[2], err, errlen);
  if (rc) return rc;
  RQA_CUDA(cudaEventRecord(ws->ev[3], st), "event");
  rc = copy_out(ws, ws->hist, hn, flags, diag, vert, white, points, mismatches, st, err, errlen);
  if (rc) return rc;
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
    timing[8] = p.var.prec == 2 ? 2.0 : (double)p.filt;
    timing[9] = (double)p.band32;
    timing[10] = p.cand;
  }
  return RQA_OK;
}

int rqa_run_multi(const double* series, int64_t len, int32_t m, int32_t tau, int32_t metric,
                  double radius, int64_t theiler, int32_t precision, const int32_t* devices,
                  int32_t n_devices, int32_t flags, int64_t* diag, int64_t* vert, int64_t* white,
                  int64_t* points, int64_t* mismatches, double* timing, char* err,
                  size_t errlen) {
  NvtxRange nvtx_("rqa_run_multi");
  if (!series || !diag || !vert || !white || !points || !devices)
    return set_err(err, errlen, "null pointer argument"), RQA_EINVAL;
  if (precision != 64 && precision != 32)
    return set_err(err, errlen, "precision must be 64 or 32"), RQA_EINVAL;
  if (n_devices < 1 || n_devices > kMaxSlots)
    return set_err(err, errlen, "n_devices must be in [1, %d]", kMaxSlots), RQA_EINVAL;
  Problem p;
  int rc = validate(len, m, tau, metric, radius, theiler, &p, err, errlen);
  if (rc) return rc;
  p.precision = precision;
  const int ndev = rqa_device_count();
  if (ndev <= 0) return set_err(err, errlen, "no CUDA device available"), RQA_EDEVICE;
  for (int g = 0; g < n_devices; ++g)
    if (devices[g] < 0 || devices[g] >= ndev || devices[g] >= kMaxDevices)
      return set_err(err, errlen, "device %d out of range (%d visible)", devices[g], ndev),
             RQA_EINVAL;
  if (n_devices == 1)
    return rqa_run_prec(series, len, m, tau, metric, radius, theiler, precision, devices[0],
                        flags, diag, vert, white, points, mismatches, timing, err, errlen);
  const auto t0 = std::chrono::steady_clock::now();
  const int G = n_devices;
  const std::vector<int64_t> bounds = area_stripes(p.n, G, 1024);
  std::vector<StripeJob> jobs(G);
  std::vector<std::unique_lock<std::mutex>> locks;
  for (int g = 0; g < G; ++g) {
    jobs[g].dev = devices[g];
    for (int q = 0; q < g; ++q) jobs[g].slot += devices[q] == devices[g];
    jobs[g].lo = bounds[g];
    jobs[g].hi = bounds[g + 1];
    jobs[g].ws = workspace(jobs[g].dev, jobs[g].slot);
  }
  // every workspace is locked for the whole call, in one global order (the
  // (slot, device) key): concurrent calls with permuted device lists cannot
  // deadlock
  {
    std::vector<int> order(G);
    for (int g = 0; g < G; ++g) order[g] = g;
    std::sort(order.begin(), order.end(), [&](int x, int y) {
      return jobs[x].slot * kMaxDevices + jobs[x].dev < jobs[y].slot * kMaxDevices + jobs[y].dev;
    });
    locks.reserve(G);
    for (int g : order) locks.emplace_back(jobs[g].ws->mu);
  }
  {
    std::vector<std::thread> th;
    for (int g = 0; g < G; ++g)
      th.emplace_back([&, g] { jobs[g].rc = run_stripe_job(&jobs[g], p, series); });
    for (auto& t : th) t.join();
  }
  for (int g = 0; g < G; ++g)
    if (jobs[g].rc) return set_err(err, errlen, "device %d: %s", jobs[g].dev, jobs[g].err), jobs[g].rc;

  // gather the stripe summaries and sum the histograms on the first device
  // (peer copies over NVLink; stripes already on that device are added in
  // place), stitch there, then one copy-back of the (sparse) result
  StripeJob& j0 = jobs[0];
  Workspace* ws0 = j0.ws;
  RQA_CUDA(cudaSetDevice(j0.dev), "cudaSetDevice");
  for (int g = 1; g < G; ++g)
    if (jobs[g].dev != j0.dev) {
      int can = 0;
      cudaDeviceCanAccessPeer(&can, j0.dev, jobs[g].dev);
      if (can && cudaDeviceEnablePeerAccess(jobs[g].dev, 0) != cudaSuccess) cudaGetLastError();
    }
  cudaStream_t st = ws0->stream;
  const size_t n = (size_t)p.n, hn = n + 1, hcount = 3 * hn + 2;
  // gather area: [G][n] prefix, [G][n] suffix, [G][2n] column parts, [2n] row
  // parts, then one histogram set (peer copy staging), 8-byte aligned
  const size_t sum_words = (size_t)G * 4 * n + 2 * n;
  const size_t hist_off = (sum_words + 1) & ~(size_t)1;
  RQA_CUDA(grow(&ws0->gather, &ws0->gather_cap, hist_off + 2 * hcount), "allocating gather");
  int32_t* gpre = ws0->gather;
  int32_t* gsuf = gpre + (size_t)G * n;
  uint32_t* gcol = reinterpret_cast<uint32_t*>(gsuf + (size_t)G * n);
  uint32_t* grow_ = gcol + (size_t)G * 2 * n;
  unsigned long long* stage = reinterpret_cast<unsigned long long*>(ws0->gather + hist_off);
  unsigned long long* hsum = j0.hist;  // stripe 0's histograms accumulate the others
  RQA_CUDA(cudaEventRecord(ws0->ev[3], st), "event");
  const int hblocks = (int)std::min<size_t>((hcount + 255) / 256, 148 * 8);
  for (int g = 0; g < G; ++g) {
    const StripeJob& j = jobs[g];
    if (j.hi > j.lo) {  // an empty stripe has no summaries (the stitch skips it)
      RQA_CUDA(cudaMemcpyPeerAsync(gpre + g * n, j0.dev, j.pre, j.dev, n * 4, st), "gather");
      RQA_CUDA(cudaMemcpyPeerAsync(gsuf + g * n, j0.dev, j.suf, j.dev, n * 4, st), "gather");
      RQA_CUDA(cudaMemcpyPeerAsync(gcol + g * 2 * n, j0.dev, j.col, j.dev, 2 * n * 4, st),
               "gather");
      RQA_CUDA(cudaMemcpyPeerAsync(grow_ + 2 * j.lo, j0.dev, j.row + 2 * j.lo, j.dev,
                                   (size_t)(j.hi - j.lo) * 2 * 4, st),
               "gather");
    }
    if (g == 0) continue;
    const unsigned long long* src = j.hist;
    if (j.dev != j0.dev) {
      RQA_CUDA(cudaMemcpyPeerAsync(stage, j0.dev, j.hist, j.dev, hcount * 8, st), "gather");
      src = stage;
    }
    hist_accumulate_kernel<<<hblocks, 256, 0, st>>>(hsum, src, (int64_t)hcount);
    RQA_CUDA(cudaGetLastError(), "launching histogram reduction");
    g_launches++;
  }
  rc = stitch_stripes(ws0, gpre, gsuf, gcol, grow_, bounds.data(), G, p.n, hsum, st, err, errlen);
  if (rc) return rc;
  RQA_CUDA(cudaEventRecord(ws0->ev[4], st), "event");
  rc = copy_out(ws0, hsum, hn, flags, diag, vert, white, points, mismatches, st, err, errlen);
  if (rc) return rc;
  if (timing) {
    float stitch_ms = 0.f, kern_ms = 0.f;
    cudaEventElapsedTime(&stitch_ms, ws0->ev[3], ws0->ev[4]);
    for (const auto& j : jobs) kern_ms = std::max(kern_ms, j.ms);
    const double wall =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (int q = 0; q < RQA_TIMING_SLOTS; ++q) timing[q] = 0.0;
    timing[1] = kern_ms * 1e-3;
    timing[2] = stitch_ms * 1e-3;
    timing[4] = wall;
    timing[5] = wall > 0 ? (double)p.n * (double)p.n / wall : 0.0;
    timing[6] = (double)j0.var.band_rows();
    timing[7] = (double)G;
    timing[8] = j0.var.prec == 2 ? 2.0 : (double)j0.filt;
    timing[9] = (double)j0.band32;
    timing[10] = j0.cand;
  }
  return RQA_OK;
}

int rqa_run(const double* series, int64_t len, int32_t m, int32_t tau, int32_t metric,
            double radius, int64_t theiler, int32_t device, int64_t* diag, int64_t* vert,
            int64_t* white, int64_t* points, double* timing, char* err, size_t errlen) {
  return rqa_run_prec(series, len, m, tau, metric, radius, theiler, 64, device, 0, diag, vert,
                      white, points, nullptr, timing, err, errlen);
}

int rqa_run_device_prec(const double* d_series, int64_t len, int32_t m, int32_t tau,
                        int32_t metric, double radius, int64_t theiler, int32_t precision,
                        int64_t row_lo, int64_t row_hi, int32_t mode, int64_t* d_hist,
                        int64_t* d_points, int64_t* d_mismatches, int32_t* d_stripe_prefix,
                        int32_t* d_stripe_suffix, uint32_t* d_stripe_col, uint32_t* d_rowlead,
                        void* stream, char* err, size_t errlen) {
  NvtxRange nvtx_("rqa_run_device");
  if (!d_series || !d_hist || !d_points)
    return set_err(err, errlen, "null pointer argument"), RQA_EINVAL;
  if (precision != 64 && precision != 32)
    return set_err(err, errlen, "precision must be 64 or 32"), RQA_EINVAL;
  if (precision == 32 && !d_mismatches)
    return set_err(err, errlen, "fp32 mode needs a mismatch counter"), RQA_EINVAL;
  Problem p;
  int rc = validate(len, m, tau, metric, radius, theiler, &p, err, errlen);
  if (rc) return rc;
  p.precision = precision;
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
  rc = plan_precision(ws, &p, st, err, errlen);
  if (!rc) rc = plan_prefilter(ws, &p, st, err, errlen);
  if (rc) return rc;
  if (p.filt == 0 && !d_mismatches) {  // exact filter: counter unused but must exist
    RQA_CUDA(grow(&ws->maxbits, &ws->maxbits_cap, 1), "allocating");
    p.mism = ws->maxbits;
  } else {
    p.mism = reinterpret_cast<unsigned long long*>(d_mismatches);
  }
  if (mode == kFoldFinal)
    return run_full(ws, p, reinterpret_cast<unsigned long long*>(d_hist),
                    reinterpret_cast<unsigned long long*>(d_points), st, nullptr, err, errlen);
  return launch_rows(ws, p, row_lo, row_hi, mode, reinterpret_cast<unsigned long long*>(d_hist),
                     reinterpret_cast<unsigned long long*>(d_points), d_stripe_prefix,
                     d_stripe_suffix, d_stripe_col, d_rowlead, st, nullptr, err, errlen);
}

int rqa_run_device(const double* d_series, int64_t len, int32_t m, int32_t tau, int32_t metric,
                   double radius, int64_t theiler, int64_t row_lo, int64_t row_hi, int32_t mode,
                   int64_t* d_hist, int64_t* d_points, int32_t* d_stripe_prefix,
                   int32_t* d_stripe_suffix, uint32_t* d_stripe_col, uint32_t* d_rowlead,
                   void* stream, char* err, size_t errlen) {
  return rqa_run_device_prec(d_series, len, m, tau, metric, radius, theiler, 64, row_lo, row_hi,
                             mode, d_hist, d_points, nullptr, d_stripe_prefix, d_stripe_suffix,
                             d_stripe_col, d_rowlead, stream, err, errlen);
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
    cudaSetDevice((int)(d % kMaxDevices));
    cudaFree(ws->gather);
    cudaFree(ws->bins);
    cudaFree(ws->s_pad);
    cudaFree(ws->sf_pad);
    cudaFree(ws->maxbits);
    cudaFree(ws->stats);
    if (ws->host_stats) cudaFreeHost(ws->host_stats);
    cudaFree(ws->ps);
    cudaFree(ws->cs);
    cudaFree(ws->rowlead);
    cudaFree(ws->rowpiece);
    cudaFree(ws->drec);
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
