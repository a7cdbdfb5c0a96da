// rqa_tiles.cu -- the reference's per-tile operator API on the GPU.
//
// tiledrqa exposes its engine as operators over materialised tiles
// (engine.py:55-212): create_recurrence_matrix fills a tile's packed bits,
// detect_diagonal_lines / detect_vertical_lines scan them with carry-over
// buffers, flush_carryovers closes the open runs.  run_analysis never uses
// these on the B200 (the fused kernel never materialises a tile), but callers
// that drive the operators themselves get them here: rqa_block builds the
// bits (rqa_plot.cu) and rqa_tile_scan runs the scans, one thread per matrix
// diagonal / column of the tile, with the carry contract of _combine_runs
// (engine.py:287-319) in its sequential form: a run starting at the segment
// start absorbs the carry, a carry with no run at the segment start is
// counted ("stale"), runs ending inside are counted at their absorbed
// length, a run touching the segment end is written back as the new carry.
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <mutex>
#include <vector>

#include "../../include/rqa_b200.h"

namespace rqa {
void note_launch();
}

namespace {

void tile_err(char* err, size_t errlen, const char* fmt, ...) {
  if (!err || errlen == 0) return;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(err, errlen, fmt, ap);
  va_end(ap);
}

// bit (u, v) of an h x w tile packed row-major, MSB first (np.packbits of the
// flattened block, engine.py:163)
__device__ __forceinline__ int tile_bit(const uint8_t* bits, int64_t w, int64_t u, int64_t v) {
  const int64_t q = u * w + v;
  return (bits[q >> 3] >> (7 - (int)(q & 7))) & 1;
}

// Sequential _combine_runs over one segment: `want` selects runs of ones or
// zeroes; lengths that reach the histogram are < nbins by construction.
__device__ __forceinline__ void scan_seq(const uint8_t* bits, int64_t w, int64_t u0, int64_t v0,
                                         int64_t du, int64_t dv, int64_t len, int want,
                                         long long* carry, unsigned long long* hist) {
  long long run = *carry;
  for (int64_t q = 0; q < len; ++q) {
    if (tile_bit(bits, w, u0 + q * du, v0 + q * dv) == want) {
      ++run;
    } else if (run > 0) {
      atomicAdd(&hist[run], 1ull);
      run = 0;
    }
  }
  *carry = run;
}

// kind 0: diagonals o = v - u in [-(h-1), w-1] (engine.py:398-433);
// kind 1: columns, runs of ones and of zeroes (engine.py:338-361).
__global__ void tile_scan_kernel(const uint8_t* bits, int64_t h, int64_t w, int kind,
                                 long long* carry_a, long long* carry_b,
                                 unsigned long long* hist_a, unsigned long long* hist_b) {
  const int64_t nseq = kind == 0 ? h + w - 1 : w;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nseq;
       s += (int64_t)gridDim.x * blockDim.x) {
    if (kind == 0) {
      const int64_t o = s - (h - 1);
      const int64_t u0 = o < 0 ? -o : 0;
      const int64_t u1 = h < w - o ? h : w - o;
      scan_seq(bits, w, u0, u0 + o, 1, 1, u1 - u0, 1, &carry_a[s], hist_a);
    } else {
      scan_seq(bits, w, 0, s, 1, 0, h, 1, &carry_a[s], hist_a);
      scan_seq(bits, w, 0, s, 1, 0, h, 0, &carry_b[s], hist_b);
    }
  }
}

struct TileWs {
  std::mutex mu;
  uint8_t* bits = nullptr;
  size_t bits_cap = 0;
  long long* carry = nullptr;
  size_t carry_cap = 0;
  unsigned long long* hist = nullptr;
  size_t hist_cap = 0;
};

TileWs g_tile_ws[64];

template <typename T>
cudaError_t grow_buf(T** p, size_t* cap, size_t need) {
  if (*cap >= need) return cudaSuccess;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), need * sizeof(T));
  if (e == cudaSuccess) *cap = need;
  return e;
}

}  // namespace

extern "C" int rqa_tile_scan(const uint8_t* tile_bits, int64_t height, int64_t width, int64_t n,
                             int32_t kind, int64_t* carry_a, int64_t* carry_b, int64_t* hist_a,
                             int64_t* hist_b, int32_t device, char* err, size_t errlen) {
  if (!tile_bits || !carry_a || !hist_a || (kind == 1 && (!carry_b || !hist_b)))
    return tile_err(err, errlen, "null pointer argument"), RQA_EINVAL;
  if (height < 1 || width < 1 || n < 1 || height > n || width > n || (kind != 0 && kind != 1))
    return tile_err(err, errlen, "invalid tile geometry or kind"), RQA_EINVAL;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= 0) {
    cudaGetLastError();
    return tile_err(err, errlen, "no CUDA device available"), RQA_EDEVICE;
  }
  if (device < 0 || device >= ndev || device >= 64)
    return tile_err(err, errlen, "device %d out of range", device), RQA_EINVAL;
  TileWs& ws = g_tile_ws[device];
  std::lock_guard<std::mutex> lk(ws.mu);
  const int64_t nseq = kind == 0 ? height + width - 1 : width;
  const int nbuf = kind == 0 ? 1 : 2;
  // longest possible closed run: carried length + the segment
  long long cmax = 0;
  for (int64_t q = 0; q < nseq; ++q) {
    cmax = std::max<long long>(cmax, carry_a[q]);
    if (kind == 1) cmax = std::max<long long>(cmax, carry_b[q]);
  }
  if (cmax < 0) return tile_err(err, errlen, "negative carry-over"), RQA_EINVAL;
  const size_t nbins = (size_t)(cmax + std::max(height, width) + 1);
  const size_t nbytes = (size_t)((height * width + 7) / 8);
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = grow_buf(&ws.bits, &ws.bits_cap, nbytes);
  if (e == cudaSuccess) e = grow_buf(&ws.carry, &ws.carry_cap, (size_t)nbuf * nseq);
  if (e == cudaSuccess) e = grow_buf(&ws.hist, &ws.hist_cap, (size_t)nbuf * nbins);
  if (e == cudaSuccess) e = cudaMemcpy(ws.bits, tile_bits, nbytes, cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaMemcpy(ws.carry, carry_a, nseq * sizeof(long long), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && kind == 1)
    e = cudaMemcpy(ws.carry + nseq, carry_b, nseq * sizeof(long long), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(ws.hist, 0, (size_t)nbuf * nbins * sizeof(unsigned long long));
  if (e != cudaSuccess) return tile_err(err, errlen, "tile scan setup: %s", cudaGetErrorString(e)), RQA_EDEVICE;
  const int threads = 256;
  const int blocks = (int)std::min<int64_t>((nseq + threads - 1) / threads, 148 * 8);
  tile_scan_kernel<<<blocks, threads>>>(ws.bits, height, width, kind, ws.carry, ws.carry + nseq,
                                        ws.hist, ws.hist + nbins);
  rqa::note_launch();
  e = cudaGetLastError();
  std::vector<unsigned long long> h((size_t)nbuf * nbins);
  if (e == cudaSuccess)
    e = cudaMemcpy(h.data(), ws.hist, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess)
    e = cudaMemcpy(carry_a, ws.carry, nseq * sizeof(long long), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && kind == 1)
    e = cudaMemcpy(carry_b, ws.carry + nseq, nseq * sizeof(long long), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return tile_err(err, errlen, "tile scan: %s", cudaGetErrorString(e)), RQA_EDEVICE;
  // hist_a / hist_b hold n+1 bins (LineHistograms); nbins <= n + 1 always
  const size_t lim = std::min<size_t>(nbins, (size_t)n + 1);
  for (size_t q = 0; q < lim; ++q) {
    hist_a[q] += (int64_t)h[q];
    if (kind == 1) hist_b[q] += (int64_t)h[nbins + q];
  }
  return RQA_OK;
}
