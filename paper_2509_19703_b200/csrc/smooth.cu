// smooth.cu -- K5: smooth-kNN rho / sigma / directed weights (float64).
//
// Replaces neighbors.py:261-318 (smooth_knn_weights up to the weight matrix),
// /root/reference/pkg/src/graph_umap/neighbors.py.  One thread per row,
// following the vectorised numpy control flow row by row:
//   rho = min over the row (rows padded to kmax with +inf)
//   all_equal rows          -> sigma = 1e3
//   s(1e3) < target         -> sigma = 1e3 ; s(1e-3) > target -> sigma = 1e-3
//   else 64 bisection steps on [1e-3, 1e3], stop when |s - target| < 1e-5,
//   s > target -> hi = mid else lo = mid, rows still live after 64 steps take
//   the next midpoint.
// s(sigma) is numpy's row sum of exp(-(d - rho) / sigma) over the kmax-wide
// padded row, in numpy's pairwise_sum order (8 accumulators, tree combine,
// sequential tail; halves above 128).  Compiled with -fmad=false so every
// float64 operation rounds as in numpy.
#include <cmath>

#include "common.cuh"
#include "gumap.h"

namespace gu {
namespace {

// x(i) = exp(-(d_i - rho) / sigma), or 0 past the row.  Rows come sorted by
// (distance, id), so a run of equal distances reuses the last value: the same
// float64 expression on the same operands, i.e. bit-identical, with one exp
// per distinct distance (2-3 per row on hop distances) instead of k.
struct RowView {
  const int* d;
  int c;
  double rho;
  double sigma;
  int last_d;
  double last_v;
  __device__ __forceinline__ void set_sigma(double s) {
    sigma = s;
    last_d = -1;  // hop distances are >= 0
  }
  __device__ __forceinline__ double x(int i) {
    if (i >= c) return 0.0;
    const int di = d[i];
    if (di != last_d) {
      last_d = di;
      last_v = exp(-((double)di - rho) / sigma);
    }
    return last_v;
  }
};

__device__ double pairwise(RowView& r, int start, int len) {
  if (len < 8) {
    double res = 0.;
    for (int i = 0; i < len; i++) res += r.x(start + i);
    return res;
  } else if (len <= 128) {
    double a0 = r.x(start + 0), a1 = r.x(start + 1), a2 = r.x(start + 2), a3 = r.x(start + 3);
    double a4 = r.x(start + 4), a5 = r.x(start + 5), a6 = r.x(start + 6), a7 = r.x(start + 7);
    int i;
    for (i = 8; i < len - (len % 8); i += 8) {
      a0 += r.x(start + i + 0);
      a1 += r.x(start + i + 1);
      a2 += r.x(start + i + 2);
      a3 += r.x(start + i + 3);
      a4 += r.x(start + i + 4);
      a5 += r.x(start + i + 5);
      a6 += r.x(start + i + 6);
      a7 += r.x(start + i + 7);
    }
    double res = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
    for (; i < len; i++) res += r.x(start + i);
    return res;
  } else {
    int n2 = len / 2;
    n2 -= n2 % 8;
    return pairwise(r, start, n2) + pairwise(r, start + n2, len - n2);
  }
}

__global__ void __launch_bounds__(128)
    smooth_kernel(long long n, const long long* __restrict__ indptr, const int* __restrict__ dist,
                  int kmax, double target, double* __restrict__ rho_out,
                  double* __restrict__ sigma_out, double* __restrict__ w_out) {
  const double SMIN = 1e-3, SMAX = 1e3, TOL = 1e-5;
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (long long)gridDim.x * blockDim.x) {
    const long long lo = indptr[v];
    const int c = (int)(indptr[v + 1] - lo);
    RowView r;
    r.d = dist + lo;
    r.c = c < kmax ? c : kmax;
    double rho = INFINITY;
    for (int i = 0; i < r.c; i++) rho = fmin(rho, (double)r.d[i]);
    bool all_equal = true;
    for (int i = 0; i < r.c; i++)
      if ((double)r.d[i] != rho) all_equal = false;
    r.rho = rho;
    double sigma = SMAX;
    if (!all_equal) {
      r.set_sigma(SMAX);
      const double s_hi = pairwise(r, 0, kmax);
      r.set_sigma(SMIN);
      const double s_lo = pairwise(r, 0, kmax);
      const bool clamp_hi = s_hi < target, clamp_lo = s_lo > target;
      if (clamp_hi) sigma = SMAX;
      if (clamp_lo) sigma = SMIN;
      if (!clamp_hi && !clamp_lo) {
        double los = SMIN, his = SMAX, mid = (los + his) / 2.0;
        bool live = true;
        for (int it = 0; it < 64; it++) {
          r.set_sigma(mid);
          const double s = pairwise(r, 0, kmax);
          if (fabs(s - target) < TOL) {
            sigma = mid;
            live = false;
            break;
          }
          if (s > target) his = mid; else los = mid;
          mid = (los + his) / 2.0;
        }
        if (live) sigma = mid;
      }
    }
    rho_out[v] = rho;
    sigma_out[v] = sigma;
    if (w_out)
      for (int i = 0; i < c; i++) w_out[lo + i] = exp(-((double)r.d[i] - rho) / sigma);
  }
}

}  // namespace
}  // namespace gu

using namespace gu;

extern "C" int gu_smooth_knn(int64_t n, const int64_t* indptr, const int32_t* dist, int32_t kmax,
                             double target, double* rho, double* sigma, double* w, void* stream) {
  if (n < 0 || kmax < 1) {
    set_error("gu_smooth_knn: bad arguments (n=%lld kmax=%d)", (long long)n, kmax);
    return GU_ERR_ARG;
  }
  if (n == 0) return GU_OK;
  long long blocks = (n + 127) / 128;
  if (blocks > 148LL * 32) blocks = 148LL * 32;
  smooth_kernel<<<(unsigned)blocks, 128, 0, (cudaStream_t)stream>>>(
      n, (const long long*)indptr, dist, kmax, target, rho, sigma, w);
  GU_CHECK_LAUNCH("smooth_kernel");
  return GU_OK;
}
