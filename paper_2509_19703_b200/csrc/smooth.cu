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

// sigma of one row (the reference's control flow, see the file header);
// rho_out receives the row minimum
__device__ double row_sigma(const int* d, int c, int kmax, double target, double* rho_out) {
  const double SMIN = 1e-3, SMAX = 1e3, TOL = 1e-5;
  RowView r;
  r.d = d;
  r.c = c < kmax ? c : kmax;
  double rho = INFINITY;
  for (int i = 0; i < r.c; i++) rho = fmin(rho, (double)r.d[i]);
  bool all_equal = true;
  for (int i = 0; i < r.c; i++)
    if ((double)r.d[i] != rho) all_equal = false;
  r.rho = rho;
  *rho_out = rho;
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
  return sigma;
}

// ---- memoised sigma.  A row's sigma is a function of its padded distance
// vector alone, and rows arrive sorted by (distance, id), so the vector is
// its run-length profile (distance, count) per run.  kNN rows of hop
// distances have a handful of profiles (c5: 4M rows, ~10^2 profiles), so the
// bisection runs once per profile: rows are keyed (<= 4 runs, distance < 256,
// count < 64), the keys deduplicated into a device table, sigma solved per
// table entry on a representative row, and every row reads it back.  Rows
// that do not fit a key, or find the table full, are solved directly.  The
// result is the same float64 computation on the same operands: bit-identical.
// (SigTable and its constants live in common.cuh: symmetrize.cu reads the
// per-run weights back through memo_weight)
__device__ __forceinline__ unsigned long long sig_mix(unsigned long long x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  return x;
}

// 64-bit profile key (bit 63 marks a key; 0 = none): up to 4 runs of 14 bits
__device__ __forceinline__ unsigned long long row_key(const int* d, int c) {
  unsigned long long key = 1ull << 63;
  int runs = 0, i = 0;
  while (i < c) {
    const int di = d[i];
    int j = i + 1;
    while (j < c && d[j] == di) j++;
    const int cnt = j - i;
    if (runs == 4 || di < 0 || di > 255 || cnt > 63) return SIG_EMPTY;
    key |= (unsigned long long)((di << 6) | cnt) << (14 * runs);
    runs++;
    i = j;
  }
  return key | ((unsigned long long)runs << 56);
}

__global__ void sig_clear(SigTable* __restrict__ tab) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < SIG_TABLE; i += gridDim.x * blockDim.x)
    tab->key[i] = SIG_EMPTY;
}

// pass 1 (thread per row): key -> table slot, kept in slot_out (-1: direct)
__global__ void sig_keys(long long n, const long long* __restrict__ indptr,
                         const int* __restrict__ dist, int kmax, SigTable* __restrict__ tab,
                         int* __restrict__ slot_out) {
  const int lane = threadIdx.x & 31;
  for (long long base = (long long)blockIdx.x * blockDim.x + threadIdx.x - lane; base < n;
       base += (long long)gridDim.x * blockDim.x) {
    const long long v = base + lane;
    unsigned long long key = SIG_EMPTY;
    if (v < n) {
      const long long lo = indptr[v];
      const int c = (int)(indptr[v + 1] - lo);
      if (c <= kmax) key = row_key(dist + lo, c);
    }
    // one table lookup per distinct key of the warp
    const unsigned grp = __match_any_sync(0xffffffffu, key);
    const int leader = __ffs(grp) - 1;
    int slot = -1;
    if (lane == leader && key != SIG_EMPTY) {
      unsigned h = (unsigned)sig_mix(key) & (SIG_TABLE - 1);
      for (int probe = 0; probe < SIG_TABLE; probe++) {
        unsigned long long cur = *(volatile unsigned long long*)&tab->key[h];
        if (cur == SIG_EMPTY) {
          cur = atomicCAS(&tab->key[h], SIG_EMPTY, key);
          if (cur == SIG_EMPTY) {  // inserted: this row represents the profile
            tab->rep[h] = v;
            slot = (int)h;
            break;
          }
        }
        if (cur == key) {
          slot = (int)h;
          break;
        }
        h = (h + 1) & (SIG_TABLE - 1);
      }
    }
    slot = __shfl_sync(0xffffffffu, slot, leader);
    if (v < n) slot_out[v] = slot;
  }
}

// pass 2 (thread per table entry): sigma of each profile on its representative
__global__ void sig_solve(const long long* __restrict__ indptr, const int* __restrict__ dist,
                          int kmax, double target, SigTable* __restrict__ tab) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < SIG_TABLE; s += gridDim.x * blockDim.x) {
    if (tab->key[s] == SIG_EMPTY) continue;
    const long long v = tab->rep[s];
    const long long lo = indptr[v];
    double rho;
    const int c = (int)(indptr[v + 1] - lo);
    const double sigma = row_sigma(dist + lo, c, kmax, target, &rho);
    tab->val[s] = sigma;
    tab->rho[s] = rho;
    // per-run weights: the same expression the per-entry path evaluates
    const unsigned long long key = tab->key[s];
    const int runs = (int)((key >> 56) & 7);
    unsigned ends = 0;
    int end = 0;
    for (int j = 0; j < 4; j++) {
      if (j < runs) {
        const int dj = (int)((key >> (14 * j + 6)) & 255);
        end += (int)((key >> (14 * j)) & 63);
        tab->w[s][j] = exp(-((double)dj - rho) / sigma);
      }
      ends |= (unsigned)(j < runs ? end : 255) << (8 * j);
    }
    tab->ends[s] = ends;
  }
}

// pass 3 (warp per 32 consecutive rows): lane l takes row base + l's rho and
// sigma (table, or solved directly), then the warp writes the weights of the
// 32 rows' entries coalesced, each entry finding its row among the lanes by
// a shuffle search; w = exp(-(d - rho) / sigma) as in the reference
__global__ void __launch_bounds__(128)
    smooth_kernel(long long n, const long long* __restrict__ indptr, const int* __restrict__ dist,
                  int kmax, double target, const SigTable* __restrict__ tab,
                  const int* __restrict__ slot_in, double* __restrict__ rho_out,
                  double* __restrict__ sigma_out, double* __restrict__ w_out) {
  const int lane = threadIdx.x & 31;
  for (long long base = (long long)blockIdx.x * blockDim.x + threadIdx.x - lane; base < n;
       base += (long long)gridDim.x * blockDim.x) {
    const long long v = base + lane;
    const bool valid = v < n;
    const long long lo = valid ? indptr[v] : 0;
    const long long hi = valid ? indptr[v + 1] : 0;
    double rho = 0.0, sigma = 0.0;
    const int slot = valid && slot_in ? slot_in[v] : -1;
    if (valid) {
      if (slot >= 0) {
        rho = tab->rho[slot];
        sigma = tab->val[slot];
      } else {
        sigma = row_sigma(dist + lo, (int)(hi - lo), kmax, target, &rho);
      }
      rho_out[v] = rho;
      sigma_out[v] = sigma;
    }
    if (!w_out) continue;
    const int nv = (int)min(32LL, n - base);  // valid lanes
    const long long e0 = __shfl_sync(0xffffffffu, lo, 0);
    const long long e1 = __shfl_sync(0xffffffffu, hi, nv - 1);
    for (long long eb = e0; eb < e1; eb += 32) {
      const long long e = eb + lane;
      int l = 0;  // last lane whose row starts at or before e
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const long long s0 = __shfl_sync(0xffffffffu, lo, (l + step) & 31);
        if (l + step < nv && s0 <= e) l += step;
      }
      const int r_slot = __shfl_sync(0xffffffffu, slot, l);
      const long long r_lo = __shfl_sync(0xffffffffu, lo, l);
      const double r_rho = __shfl_sync(0xffffffffu, rho, l);
      const double r_sig = __shfl_sync(0xffffffffu, sigma, l);
      if (e < e1) {
        double w;
        if (r_slot >= 0) {  // profiled row: its run's precomputed weight
          w = memo_weight(tab, r_slot, (unsigned)(e - r_lo));
        } else {
          w = exp(-((double)dist[e] - r_rho) / r_sig);
        }
        w_out[e] = w;
      }
    }
  }
}

}  // namespace
}  // namespace gu

using namespace gu;

// memoised-sigma scratch: the profile table + one slot per row (rows below
// SMOOTH_MEMO_MIN_ROWS are solved directly and need no workspace)
constexpr long long SMOOTH_MEMO_MIN_ROWS = 4096;

extern "C" size_t gu_smooth_knn_workspace_size(int64_t n) {
  if (n < SMOOTH_MEMO_MIN_ROWS) return 0;
  return SIG_TABLE_BYTES + sizeof(int) * (size_t)n;
}

extern "C" int gu_smooth_knn(int64_t n, const int64_t* indptr, const int32_t* dist, int32_t kmax,
                             double target, double* rho, double* sigma, double* w,
                             void* workspace, size_t ws_bytes, void* stream) {
  if (n < 0 || kmax < 1) {
    set_error("gu_smooth_knn: bad arguments (n=%lld kmax=%d)", (long long)n, kmax);
    return GU_ERR_ARG;
  }
  if (n == 0) return GU_OK;
  cudaStream_t st = (cudaStream_t)stream;
  long long blocks = (n + 127) / 128;
  if (blocks > 148LL * 32) blocks = 148LL * 32;
  const size_t need = gu_smooth_knn_workspace_size(n);
  if (need && (!workspace || ws_bytes < need)) {
    set_error("gu_smooth_knn: workspace %zu < %zu bytes", ws_bytes, need);
    return GU_ERR_WORKSPACE;
  }
  SigTable* tab = need ? (SigTable*)workspace : nullptr;
  int* slots = need ? (int*)((char*)workspace + SIG_TABLE_BYTES)
                    : nullptr;
  if (slots) {
    sig_clear<<<8, 256, 0, st>>>(tab);
    GU_CHECK_LAUNCH("sig_clear");
    sig_keys<<<(unsigned)blocks, 128, 0, st>>>(n, (const long long*)indptr, dist, kmax, tab,
                                                slots);
    GU_CHECK_LAUNCH("sig_keys");
    sig_solve<<<SIG_TABLE / 128, 128, 0, st>>>((const long long*)indptr, dist, kmax, target, tab);
    GU_CHECK_LAUNCH("sig_solve");
  }
  smooth_kernel<<<(unsigned)blocks, 128, 0, st>>>(n, (const long long*)indptr, dist, kmax, target,
                                                  tab, slots, rho, sigma, w);
  GU_CHECK_LAUNCH("smooth_kernel");
  return GU_OK;
}
