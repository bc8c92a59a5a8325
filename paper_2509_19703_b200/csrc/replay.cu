// replay.cu -- K8: order-faithful float64 replay of one sgd_sweep.
//
// Parity check (b) of the north star: replays /root/reference/pkg/src/
// graph_umap/_kernels.py:158-223 for a supplied visit order (visit_log,
// layout.py:356-357) and the accepted negatives / thetas of that sweep, in
// float64 with the reference's operation order (-fmad=false: no FMA).
//
// Visits are grouped into conflict-free waves on the host
// (gu_replay_schedule): visit i reads {u, v, c_1..c_nneg} and writes {u, v};
// wave(i) = 1 + max(last write wave of anything it touches, last read wave of
// what it writes).  Inside a wave no two visits share a written vertex or
// read a vertex another writes, so applying waves in order reproduces the
// sequential sweep exactly; a single CTA walks the waves with one
// __syncthreads per wave (the measured parallelism is ~50-500 visits/wave).
#include <cmath>
#include <vector>

#include "common.cuh"
#include "gumap.h"

namespace gu {
namespace {

__device__ __forceinline__ double clip4d(double x) {
  if (x > 4.0) return 4.0;
  if (x < -4.0) return -4.0;
  return x;
}

__global__ void __launch_bounds__(1024)
    replay_kernel(double* __restrict__ xy, const int* __restrict__ e_src,
                  const int* __restrict__ e_dst, const double* __restrict__ e_w,
                  const long long* __restrict__ order, const int* __restrict__ negs,
                  const double* __restrict__ thetas, int n_neg, double a, double b, double lr,
                  const long long* __restrict__ items, const long long* __restrict__ woff,
                  long long n_waves) {
  for (long long wv = 0; wv < n_waves; wv++) {
    for (long long j = woff[wv] + threadIdx.x; j < woff[wv + 1]; j += blockDim.x) {
      const long long i = items[j];
      const long long e = order[i];
      const int u = e_src[e], v = e_dst[e];
      const double h = e_w[e];
      double ux = xy[2 * u], uy = xy[2 * u + 1];
      double vx = xy[2 * v], vy = xy[2 * v + 1];
      double dx = ux - vx, dy = uy - vy;
      double d2 = dx * dx + dy * dy;
      if (d2 > 0.0) {
        double pb = pow(d2, b);
        double g = -2.0 * a * b * h * (pb / d2) / (a * pb + 1.0);
        double gx = clip4d(g * dx), gy = clip4d(g * dy);
        ux += lr * gx;
        uy += lr * gy;
        vx -= lr * gx;
        vy -= lr * gy;
        xy[2 * v] = vx;
        xy[2 * v + 1] = vy;
      }
      for (int q = 0; q < n_neg; q++) {
        const long long slot = i * n_neg + q;
        const int c = negs[slot];
        if (c < 0) continue;
        double cx = xy[2 * c], cy = xy[2 * c + 1];
        double ddx = ux - cx, ddy = uy - cy;
        double dd2 = ddx * ddx + ddy * ddy;
        double gx, gy;
        if (dd2 > 0.0) {
          double g = 2.0 * b / ((0.001 + dd2) * (a * pow(dd2, b) + 1.0));
          gx = clip4d(g * ddx);
          gy = clip4d(g * ddy);
        } else {
          double th = thetas[slot];
          gx = 4.0 * cos(th);
          gy = 4.0 * sin(th);
        }
        ux += lr * gx;
        uy += lr * gy;
      }
      xy[2 * u] = ux;
      xy[2 * u + 1] = uy;
    }
    __syncthreads();
  }
}

}  // namespace
}  // namespace gu

using namespace gu;

extern "C" int gu_replay_schedule(int64_t n, int64_t n_order, const int32_t* host_src,
                                  const int32_t* host_dst, const int64_t* host_order,
                                  const int32_t* host_negs, int32_t n_neg,
                                  int64_t* host_wave_items, int64_t* host_wave_offsets,
                                  int64_t* host_n_waves) {
  if (n <= 0 || n_order < 0 || n_neg < 0) {
    set_error("gu_replay_schedule: bad arguments");
    return GU_ERR_ARG;
  }
  std::vector<long long> lastW((size_t)n, 0), lastR((size_t)n, 0);
  std::vector<long long> wave((size_t)n_order);
  long long maxw = 0;
  for (long long i = 0; i < n_order; i++) {
    const long long e = host_order[i];
    const int u = host_src[e], v = host_dst[e];
    long long w = lastW[u];
    if (lastW[v] > w) w = lastW[v];
    if (lastR[u] > w) w = lastR[u];
    if (lastR[v] > w) w = lastR[v];
    for (int q = 0; q < n_neg; q++) {
      const int c = host_negs[i * n_neg + q];
      if (c >= 0 && lastW[c] > w) w = lastW[c];
    }
    w += 1;
    wave[i] = w;
    lastW[u] = w;
    lastW[v] = w;
    for (int q = 0; q < n_neg; q++) {
      const int c = host_negs[i * n_neg + q];
      if (c >= 0 && lastR[c] < w) lastR[c] = w;
    }
    if (w > maxw) maxw = w;
  }
  // counting sort by wave (waves are 1-based)
  std::vector<long long> cnt((size_t)maxw + 2, 0);
  for (long long i = 0; i < n_order; i++) cnt[(size_t)wave[i]]++;
  host_wave_offsets[0] = 0;
  for (long long w = 1; w <= maxw; w++) host_wave_offsets[w] = host_wave_offsets[w - 1] + cnt[(size_t)w];
  std::vector<long long> cur(host_wave_offsets, host_wave_offsets + maxw);
  for (long long i = 0; i < n_order; i++) host_wave_items[cur[(size_t)(wave[i] - 1)]++] = i;
  *host_n_waves = maxw;
  return GU_OK;
}

extern "C" int gu_sgd_replay_f64(int64_t n, double* coords, const int32_t* e_src,
                                 const int32_t* e_dst, const double* e_w, const int64_t* order,
                                 const int32_t* negs, const double* thetas, int32_t n_neg,
                                 double a, double b, double lr, const int64_t* wave_items,
                                 const int64_t* wave_offsets, int64_t n_waves, void* stream) {
  if (n <= 0 || n_waves < 0) {
    set_error("gu_sgd_replay_f64: bad arguments");
    return GU_ERR_ARG;
  }
  if (n_waves == 0) return GU_OK;
  replay_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(
      coords, e_src, e_dst, e_w, (const long long*)order, negs, thetas, n_neg, a, b, lr,
      (const long long*)wave_items, (const long long*)wave_offsets, n_waves);
  GU_CHECK_LAUNCH("replay_kernel");
  return GU_OK;
}
