// rqa_plot.cu -- recurrence-matrix blocks and OR-reduced recurrence plots.
//
// Device counterpart of the reference's recurrence_block (embedding.py:115-171)
// and compute_plot / _or_reduce (plotting.py:48-109): every pixel (u, v) of a
// reduction factor b is the OR of the b x b cells (i, j) with
// i in [row0 + u*b, ...), j in [col0 + v*b, ...), each cell evaluated with the
// reference's arithmetic (same operation order, no FMA, exact sqrt-free L2
// threshold, Linf as AND of component tests).  Output rows are packed
// MSB-first and padded to a byte, i.e. numpy.packbits(axis=1) / PBM raster.
#include <algorithm>
#include <cstdint>
#include <cstdio>

#include "../../include/rqa_b200.h"
#include "rqa_device.cuh"

namespace rqa {

void note_launch();  // rqa_capi.cu

struct PlotArgs {
  const double* s;
  int64_t n, row0, row1, col0, col1;
  int m, tau, metric;
  double thr;
  int64_t theiler;
  int64_t factor, rows_out, cols_out, row_bytes;
  uint8_t* out;
};

__device__ __forceinline__ bool cell(const PlotArgs& a, int64_t i, int64_t j) {
  const int64_t dij = i > j ? i - j : j - i;
  if (dij < a.theiler) return false;
  const double* ri = a.s + i;
  const double* cj = a.s + j;
  if (a.metric == kLinf || a.m == 1) {
    bool hit = true;
    for (int k = 0; k < a.m; ++k)
      hit &= fabs(__dsub_rn(ri[(int64_t)k * a.tau], cj[(int64_t)k * a.tau])) <= a.thr;
    return hit;
  }
  double acc = 0.0;
  for (int k = 0; k < a.m; ++k) {
    const double d = __dsub_rn(ri[(int64_t)k * a.tau], cj[(int64_t)k * a.tau]);
    const double t = (a.metric == kL2) ? __dmul_rn(d, d) : fabs(d);
    acc = (k == 0) ? t : __dadd_rn(acc, t);
  }
  return acc <= a.thr;
}

__global__ void plot_kernel(const PlotArgs a) {
  const int64_t total = a.rows_out * a.row_bytes;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = q / a.row_bytes, byte = q % a.row_bytes;
    const int64_t i_lo = a.row0 + u * a.factor, i_hi = min(i_lo + a.factor, a.row1);
    uint32_t bits = 0;
    for (int p = 0; p < 8; ++p) {
      const int64_t v = byte * 8 + p;
      if (v >= a.cols_out) break;
      const int64_t j_lo = a.col0 + v * a.factor, j_hi = min(j_lo + a.factor, a.col1);
      bool on = false;
      for (int64_t i = i_lo; i < i_hi && !on; ++i)
        for (int64_t j = j_lo; j < j_hi && !on; ++j) on = cell(a, i, j);
      if (on) bits |= 0x80u >> p;
    }
    a.out[q] = (uint8_t)bits;
  }
}

}  // namespace rqa

using namespace rqa;

namespace {
double l2_thr(double eps) {
  double t;
  rqa_threshold(kL2, 2, eps, &t);
  return t;
}
}  // namespace

extern "C" int rqa_block(const double* series, int64_t len, int32_t m, int32_t tau, int32_t metric,
                         double radius, int64_t theiler, int64_t row0, int64_t row1, int64_t col0,
                         int64_t col1, int32_t factor, int32_t device, uint8_t* out, char* err,
                         size_t errlen) {
  auto fail = [&](int code, const char* msg) {
    if (err && errlen) snprintf(err, errlen, "%s", msg);
    return code;
  };
  if (!series || !out) return fail(RQA_EINVAL, "null pointer argument");
  if (m < 1 || tau < 1 || metric < 0 || metric > 2 || !(radius >= 0) || theiler < 0 || factor < 1)
    return fail(RQA_EINVAL, "invalid arguments");
  const int64_t span = (int64_t)(m - 1) * tau;
  if (len <= span) return fail(RQA_ESHORT, "series too short for the embedding");
  const int64_t n = len - span;
  if (!(0 <= row0 && row0 <= row1 && row1 <= n && 0 <= col0 && col0 <= col1 && col1 <= n))
    return fail(RQA_EINVAL, "block indices out of range");
  if (rqa_device_count() <= device || device < 0) return fail(RQA_EDEVICE, "no CUDA device");
  if (cudaSetDevice(device) != cudaSuccess) return fail(RQA_EDEVICE, "cudaSetDevice failed");
  PlotArgs a;
  a.n = n;
  a.row0 = row0;
  a.row1 = row1;
  a.col0 = col0;
  a.col1 = col1;
  a.m = m;
  a.tau = tau;
  a.metric = metric;
  a.thr = (metric == kL2 && m > 1) ? l2_thr(radius) : radius;
  a.theiler = theiler;
  a.factor = factor;
  a.rows_out = (row1 - row0 + factor - 1) / factor;
  a.cols_out = (col1 - col0 + factor - 1) / factor;
  a.row_bytes = (a.cols_out + 7) / 8;
  const size_t out_bytes = (size_t)(a.rows_out * a.row_bytes);
  if (out_bytes == 0) return RQA_OK;
  double* d_s = nullptr;
  uint8_t* d_out = nullptr;
  cudaError_t e = cudaMalloc(&d_s, (size_t)len * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&d_out, out_bytes);
  if (e == cudaSuccess) e = cudaMemcpy(d_s, series, (size_t)len * sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    a.s = d_s;
    a.out = d_out;
    const int64_t blocks = std::min<int64_t>(((int64_t)out_bytes + 255) / 256, 148 * 32);
    plot_kernel<<<(int)blocks, 256>>>(a);
    e = cudaGetLastError();
    note_launch();
  }
  if (e == cudaSuccess) e = cudaMemcpy(out, d_out, out_bytes, cudaMemcpyDeviceToHost);
  cudaFree(d_s);
  cudaFree(d_out);
  if (e != cudaSuccess) {
    snprintf(err, errlen, "rqa_block: %s", cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? RQA_ENOMEM : RQA_EDEVICE;
  }
  return RQA_OK;
}
