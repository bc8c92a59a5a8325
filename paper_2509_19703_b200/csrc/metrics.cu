// metrics.cu -- layout-quality metrics on the GPU.
//
// Restates /root/reference/pkg/src/graph_umap/metrics.py:
//   stress                     metrics.py:90-132  (optimal scale, all ordered pairs)
//   count_crossings            metrics.py:135-190 + _kernels.py:244-296 (exact)
//   neighborhood_preservation  metrics.py:41-79   (r-hop ball vs |ball| nearest)
// Layout distances are scipy cdist's: sqrt(dx*dx + dy*dy) in float64 with no
// contraction (explicit _rn intrinsics; this file is also built with
// -fmad=false), so distance ties and ranks match the reference.
#include <climits>
#include <cstdio>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "common.cuh"
#include "gumap.h"

namespace gu {
namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ double cdist_xy(double2 p, double2 q) {
  const double dx = __dsub_rn(p.x, q.x), dy = __dsub_rn(p.y, q.y);
  return __dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
}

// deterministic block sum (blockDim.x a multiple of 32, <= 1024); result in
// thread 0
__device__ double block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(FULL, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); i++) r += sh[i];
  __syncthreads();
  return r;
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

struct Carve {
  char* base;
  size_t off = 0;
  template <class T>
  T* take(size_t count) {
    T* p = base ? (T*)(base + off) : nullptr;
    off = align256(off + sizeof(T) * count);
    return p;
  }
};

// ================================================================= stress
// The pair terms are accumulated inside the bitset BFS (full_bfs.cu
// MODE_STRESS): two passes over every source, no hop rows in memory.
constexpr int ST_THREADS = 256;
constexpr int ST_CTAS = 148 * 2;  // 64-source BFS batches in flight

__global__ void reduce_acc(const double2* __restrict__ acc, int nb, double2* __restrict__ out) {
  __shared__ double sh[ST_THREADS / 32];
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    a += acc[i].x;
    b += acc[i].y;
  }
  const double sa = block_sum(a, sh);
  const double sb = block_sum(b, sh);
  if (threadIdx.x == 0) *out = make_double2(sa, sb);
}

// metrics.py:112: scale = s_num / s_den if s_den > 0 else 1 (rescale off: 1)
__global__ void stress_scale(const double2* __restrict__ sums, int rescale, double* scale) {
  const double2 v = *sums;
  *scale = (rescale && v.y > 0.0) ? v.x / v.y : 1.0;
}

// out[0] = sum of the stress terms, out[1] = scale, out[2] = unreachable flag
__global__ void stress_finish(const double2* __restrict__ sums, const double* __restrict__ scale,
                              const int* __restrict__ flag, double* __restrict__ out) {
  out[0] = sums[1].x;
  out[1] = *scale;
  out[2] = (double)*flag;
}

struct StressWs {
  char* bfs;
  size_t bfs_bytes;
  double2* acc;
  double2* sums;
  double* scale;
  int* flag;
};

size_t stress_layout(long long n, char* base, StressWs* ws) {
  Carve c{base};
  StressWs w;
  w.bfs_bytes = stress_bfs_workspace(n, ST_CTAS);
  w.bfs = c.take<char>(w.bfs_bytes);
  w.acc = c.take<double2>(ST_CTAS);
  w.sums = c.take<double2>(2);
  w.scale = c.take<double>(1);
  w.flag = c.take<int>(1);
  if (ws) *ws = w;
  return c.off;
}

// ============================================================== crossings
// Exact orientation: error-free transforms + expansion sign (Shewchuk's
// orient2d, restated).  two_sum / two_diff / two_product are exact in IEEE
// double (the product through fma).
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}
__device__ __forceinline__ void two_diff(double a, double b, double& s, double& e) {
  s = __dsub_rn(a, b);
  const double bb = __dsub_rn(a, s);
  e = __dadd_rn(__dsub_rn(a, __dadd_rn(s, bb)), __dsub_rn(bb, b));
}
__device__ __forceinline__ void two_product(double a, double b, double& p, double& e) {
  p = __dmul_rn(a, b);
  e = __fma_rn(a, b, -p);
}

// sign of the exact sum of x[0..len), len <= 16: grow a nonoverlapping
// expansion term by term (zero elimination); its sign is the sign of its
// largest component, the last one
__device__ int expansion_sign(const double* x, int len) {
  double h[17];
  int hl = 0;
  for (int t = 0; t < len; t++) {
    double q = x[t];
    int k = 0;
    for (int i = 0; i < hl; i++) {
      double s, e;
      two_sum(q, h[i], s, e);
      q = s;
      if (e != 0.0) h[k++] = e;
    }
    if (q != 0.0) h[k++] = q;
    hl = k;
  }
  if (hl == 0) return 0;
  return h[hl - 1] > 0.0 ? 1 : -1;
}

// exact sign of (bx-ax)(cy-ay) - (by-ay)(cx-ax)
__device__ __noinline__ int orient_exact(double ax, double ay, double bx, double by, double cx,
                                         double cy) {
  double u1, u0, v1, v0, w1, w0, z1, z0;
  two_diff(bx, ax, u1, u0);
  two_diff(cy, ay, v1, v0);
  two_diff(by, ay, w1, w0);
  two_diff(cx, ax, z1, z0);
  double t[16];
  two_product(u1, v1, t[0], t[1]);
  two_product(u1, v0, t[2], t[3]);
  two_product(u0, v1, t[4], t[5]);
  two_product(u0, v0, t[6], t[7]);
  two_product(w1, z1, t[8], t[9]);
  two_product(w1, z0, t[10], t[11]);
  two_product(w0, z1, t[12], t[13]);
  two_product(w0, z0, t[14], t[15]);
  for (int i = 8; i < 16; i++) t[i] = -t[i];
  return expansion_sign(t, 16);
}

// float filter (ccwerrboundA = (3 + 16 eps) eps), exact fallback near zero
__device__ __forceinline__ int orient(double ax, double ay, double bx, double by, double cx,
                                      double cy) {
  const double t1 = __dmul_rn(__dsub_rn(bx, ax), __dsub_rn(cy, ay));
  const double t2 = __dmul_rn(__dsub_rn(by, ay), __dsub_rn(cx, ax));
  const double det = __dsub_rn(t1, t2);
  const double bound = 3.3306690738754716e-16 * __dadd_rn(fabs(t1), fabs(t2));
  if (det > bound) return 1;
  if (-det > bound) return -1;
  return orient_exact(ax, ay, bx, by, cx, cy);
}

// exact sign of |p - q| - |r - s| (the collinear axis choice, metrics.py:169)
__device__ int cmp_absdiff(double p, double q, double r, double s) {
  double a1, a0, b1, b0;
  two_diff(p, q, a1, a0);
  two_diff(r, s, b1, b0);
  if (a1 < 0.0 || (a1 == 0.0 && a0 < 0.0)) {
    a1 = -a1;
    a0 = -a0;
  }
  if (b1 < 0.0 || (b1 == 0.0 && b0 < 0.0)) {
    b1 = -b1;
    b0 = -b0;
  }
  const double t[4] = {a0, a1, -b0, -b1};
  return expansion_sign(t, 4);
}

// metrics.py:153-173 (+ the float filter order of _kernels.py:279-291): do
// the open segments share a point?
__device__ bool open_segments_cross(double2 p1, double2 p2, double2 p3, double2 p4) {
  const int o1 = orient(p1.x, p1.y, p2.x, p2.y, p3.x, p3.y);
  const int o2 = orient(p1.x, p1.y, p2.x, p2.y, p4.x, p4.y);
  if (o1 != 0 && o1 == o2) return false;
  const int o3 = orient(p3.x, p3.y, p4.x, p4.y, p1.x, p1.y);
  const int o4 = orient(p3.x, p3.y, p4.x, p4.y, p2.x, p2.y);
  if (o3 != 0 && o3 == o4) return false;
  if (o1 != 0 && o2 != 0 && o3 != 0 && o4 != 0) return o1 != o2 && o3 != o4;
  if (o1 == 0 && o2 == 0 && o3 == 0 && o4 == 0) {
    const bool xaxis = cmp_absdiff(p2.x, p1.x, p2.y, p1.y) >= 0;
    const double a0 = xaxis ? p1.x : p1.y, a1 = xaxis ? p2.x : p2.y;
    const double b0 = xaxis ? p3.x : p3.y, b1 = xaxis ? p4.x : p4.y;
    const double alo = fmin(a0, a1), ahi = fmax(a0, a1);
    const double blo = fmin(b0, b1), bhi = fmax(b0, b1);
    return fmax(alo, blo) < fmin(ahi, bhi);
  }
  return false;  // an endpoint on the other segment's line: not interior to both
}

// square cells of side 1/inv from (x0, y0); cell index clamped to [0, g)
struct Grid {
  double x0, y0, inv, cell;
  int g;
};

__device__ __forceinline__ int cell_of(double v, double o, double inv, int g) {
  const double f = floor(__dmul_rn(__dsub_rn(v, o), inv));
  return f < 0.0 ? 0 : (f >= (double)(g - 1) ? g - 1 : (int)f);
}

// bounding box of the coordinates -> the grid (one block)
__global__ void grid_from_bbox(const double2* __restrict__ xy, long long n, int g,
                               Grid* __restrict__ out) {
  __shared__ double sh[4][32];
  double lox = INFINITY, loy = INFINITY, hix = -INFINITY, hiy = -INFINITY;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) {
    const double2 p = xy[i];
    lox = fmin(lox, p.x);
    loy = fmin(loy, p.y);
    hix = fmax(hix, p.x);
    hiy = fmax(hiy, p.y);
  }
  for (int o = 16; o > 0; o >>= 1) {
    lox = fmin(lox, __shfl_down_sync(FULL, lox, o));
    loy = fmin(loy, __shfl_down_sync(FULL, loy, o));
    hix = fmax(hix, __shfl_down_sync(FULL, hix, o));
    hiy = fmax(hiy, __shfl_down_sync(FULL, hiy, o));
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sh[0][w] = lox;
    sh[1][w] = loy;
    sh[2][w] = hix;
    sh[3][w] = hiy;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x >> 5); i++) {
      lox = fmin(lox, sh[0][i]);
      loy = fmin(loy, sh[1][i]);
      hix = fmax(hix, sh[2][i]);
      hiy = fmax(hiy, sh[3][i]);
    }
    if (!(lox <= hix)) lox = hix = 0.0;  // n == 0
    if (!(loy <= hiy)) loy = hiy = 0.0;
    double span = fmax(hix - lox, hiy - loy);
    double cell = span > 0.0 ? span / g : 1.0;
    if (!(cell > 0.0) || !isfinite(cell)) cell = 1.0;
    *out = Grid{lox, loy, 1.0 / cell, cell, g};
  }
}

struct EdgeBox {
  double lox, loy, hix, hiy;
};

__device__ __forceinline__ EdgeBox edge_box(double2 p, double2 q) {
  return {fmin(p.x, q.x), fmin(p.y, q.y), fmax(p.x, q.x), fmax(p.y, q.y)};
}

// cells covered by each edge's bounding box: count pass (FILL = false) and
// fill pass
template <bool FILL>
__global__ void cross_raster(long long m, const int2* __restrict__ edges,
                             const double2* __restrict__ xy, const Grid* __restrict__ grid,
                             long long* __restrict__ ecount, const long long* __restrict__ eoff,
                             int* __restrict__ inc_cell, int* __restrict__ inc_edge) {
  const Grid gr = *grid;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += (long long)gridDim.x * blockDim.x) {
    const int2 uv = edges[e];
    const EdgeBox bx = edge_box(xy[uv.x], xy[uv.y]);
    const int cx0 = cell_of(bx.lox, gr.x0, gr.inv, gr.g), cx1 = cell_of(bx.hix, gr.x0, gr.inv, gr.g);
    const int cy0 = cell_of(bx.loy, gr.y0, gr.inv, gr.g), cy1 = cell_of(bx.hiy, gr.y0, gr.inv, gr.g);
    if (!FILL) {
      ecount[e] = (long long)(cx1 - cx0 + 1) * (long long)(cy1 - cy0 + 1);
    } else {
      long long o = eoff[e];
      for (int cy = cy0; cy <= cy1; cy++)
        for (int cx = cx0; cx <= cx1; cx++) {
          inc_cell[o] = cy * gr.g + cx;
          inc_edge[o] = (int)e;
          o++;
        }
    }
  }
}

// start of each cell in a cell-sorted list (lower bound); cstart[ncell] = end
__global__ void cell_starts(long long ncell, const int* __restrict__ sorted_cell,
                            long long n_inc, long long* __restrict__ cstart) {
  for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c <= ncell;
       c += (long long)gridDim.x * blockDim.x) {
    long long lo = 0, hi = n_inc;
    while (lo < hi) {
      const long long mid = (lo + hi) >> 1;
      if (sorted_cell[mid] < c) lo = mid + 1;
      else hi = mid;
    }
    cstart[c] = lo;
  }
}

__global__ void cell_pair_counts(long long ncell, const long long* __restrict__ cstart,
                                 long long* __restrict__ npairs) {
  for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < ncell;
       c += (long long)gridDim.x * blockDim.x) {
    const long long k = cstart[c + 1] - cstart[c];
    npairs[c] = k * (k - 1) / 2;
  }
}

// flattened pair index -> (cell, a < b).  A pair is judged only in the cell
// holding the lower-left corner of the two boxes' intersection, so each
// unordered pair is counted once.
__global__ void __launch_bounds__(256)
    cross_pairs(long long ncell, const long long* __restrict__ pstart,
                const long long* __restrict__ cstart, const int* __restrict__ cell_edges,
                const int2* __restrict__ edges, const double2* __restrict__ xy,
                const Grid* __restrict__ grid, unsigned long long* __restrict__ count) {
  const Grid gr = *grid;
  const long long total = pstart[ncell];
  unsigned long long mine = 0;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < total;
       p += (long long)gridDim.x * blockDim.x) {
    long long lo = 0, hi = ncell - 1;  // last c with pstart[c] <= p
    while (lo < hi) {
      const long long mid = (lo + hi + 1) >> 1;
      if (pstart[mid] <= p) lo = mid;
      else hi = mid - 1;
    }
    const long long c = lo;
    long long r = p - pstart[c];
    const long long k = cstart[c + 1] - cstart[c];
    // row a of the strict upper triangle holds pairs (a, a+1 .. k-1)
    auto row_start = [&](long long x) { return x * (2 * k - x - 1) / 2; };
    const double kk = (double)(2 * k - 1);
    double est = floor((kk - sqrt(fmax(kk * kk - 8.0 * (double)r, 0.0))) * 0.5);
    long long a = est < 0.0 ? 0 : (long long)est;
    if (a > k - 2) a = k - 2;
    while (a > 0 && row_start(a) > r) a--;
    while (a + 1 <= k - 2 && row_start(a + 1) <= r) a++;
    const long long b = a + 1 + (r - row_start(a));
    const int e1 = cell_edges[cstart[c] + a], e2 = cell_edges[cstart[c] + b];
    const int2 s = edges[e1], t = edges[e2];
    if (s.x == t.x || s.x == t.y || s.y == t.x || s.y == t.y) continue;
    const double2 p1 = xy[s.x], p2 = xy[s.y], p3 = xy[t.x], p4 = xy[t.y];
    const EdgeBox b1 = edge_box(p1, p2), b2 = edge_box(p3, p4);
    if (b2.hix < b1.lox || b2.lox > b1.hix || b2.hiy < b1.loy || b2.loy > b1.hiy) continue;
    const int ccx = cell_of(fmax(b1.lox, b2.lox), gr.x0, gr.inv, gr.g);
    const int ccy = cell_of(fmax(b1.loy, b2.loy), gr.y0, gr.inv, gr.g);
    if ((long long)ccy * gr.g + ccx != c) continue;
    if (open_segments_cross(p1, p2, p3, p4)) mine++;
  }
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_down_sync(FULL, mine, o);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(count, mine);
}

struct CrossWs {
  Grid* grid;
  long long* ecount;
  long long* eoff;
  int* inc_cell;
  int* inc_edge;
  int* sorted_cell;
  int* sorted_edge;
  long long* cstart;
  long long* pstart;
  void* tmp;
  size_t tmp_bytes;
};

size_t cross_layout(long long m, long long n_inc, int g, char* base, CrossWs* ws) {
  const long long ncell = (long long)g * g;
  size_t sort_b = 0, scan_b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sort_b, (const int*)nullptr, (int*)nullptr,
                                  (const int*)nullptr, (int*)nullptr,
                                  (int)(n_inc > 0 ? n_inc : 1));
  cub::DeviceScan::ExclusiveSum(nullptr, scan_b, (const long long*)nullptr, (long long*)nullptr,
                                (int)(m + 1 > ncell + 1 ? m + 1 : ncell + 1));
  Carve c{base};
  CrossWs w;
  w.grid = c.take<Grid>(1);
  w.ecount = c.take<long long>((size_t)m + 1);
  w.eoff = c.take<long long>((size_t)m + 1);
  w.inc_cell = c.take<int>((size_t)n_inc);
  w.inc_edge = c.take<int>((size_t)n_inc);
  w.sorted_cell = c.take<int>((size_t)n_inc);
  w.sorted_edge = c.take<int>((size_t)n_inc);
  w.cstart = c.take<long long>((size_t)ncell + 1);
  w.pstart = c.take<long long>((size_t)ncell + 1);
  w.tmp_bytes = sort_b > scan_b ? sort_b : scan_b;
  w.tmp = c.take<char>(w.tmp_bytes);
  if (ws) *ws = w;
  return c.off;
}

// ===================================================== neighborhood pres.
constexpr int NP_WARPS = 8;

// per-vertex cell ids of the drawing (same cell_of as the search)
__global__ void np_cells(const double2* __restrict__ xy, int n, const Grid* __restrict__ grid,
                         int* __restrict__ cell, int* __restrict__ ids) {
  const Grid gr = *grid;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double2 p = xy[i];
    cell[i] = cell_of(p.y, gr.y0, gr.inv, gr.g) * gr.g + cell_of(p.x, gr.x0, gr.inv, gr.g);
    ids[i] = i;
  }
}

// 64-bit key of a non-negative double distance (bit order = numeric order)
__device__ __forceinline__ unsigned long long dkey(double d) {
  return (unsigned long long)__double_as_longlong(d);
}

// One warp per vertex v (grid-stride).  hood = the r-ball of v minus v
// (metrics.py:53-64, sparse-power reachability == BFS ball), q = |hood|;
// threshold = the q-th smallest (cdist, id) key over all w != v (the stable
// argsort of metrics.py:75-76); inter = hood members at or below it.
__global__ void __launch_bounds__(NP_WARPS * 32)
    np_kernel(int n, const int* __restrict__ indptr, const int* __restrict__ indices,
              const double2* __restrict__ xy, int r, const Grid* __restrict__ grid,
              const long long* __restrict__ cstart, const int* __restrict__ cpts,
              int* __restrict__ stamps, int* __restrict__ queues, int nslots,
              const int* __restrict__ sources, int nitems, double* __restrict__ jac) {
  __shared__ unsigned hist[NP_WARPS][256];
  const Grid gr = *grid;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * NP_WARPS + warp;
  if (gw >= nslots) return;
  int* const stamp = stamps + (long long)gw * n;
  int* const queue = queues + (long long)gw * n;
  unsigned* const hh = hist[warp];
  const unsigned lt = (1u << lane) - 1u;
  for (int item = gw; item < nitems; item += nslots) {
    const int v = sources ? sources[item] : item;
    const int tag = v + 1;  // stamps start at 0; tags are unique per vertex
    if (lane == 0) stamp[v] = tag;
    __syncwarp();
    // ---- r-ball by levels; queue holds the hood in level order
    int qlen = 0, lv0 = 0, lv1 = 0;
    for (int L = 1; L <= r; L++) {
      const int pcount = (L == 1) ? 1 : lv1 - lv0;
      if (pcount == 0) break;
      const int start_len = qlen;
      for (int pi = 0; pi < pcount; pi++) {
        const int p = (L == 1) ? v : queue[lv0 + pi];
        const int b = __ldg(indptr + p), e = __ldg(indptr + p + 1);
        for (int t0 = b; t0 < e; t0 += 32) {
          const int t = t0 + lane;
          bool isnew = false;
          int w = 0;
          if (t < e) {
            w = __ldg(indices + t);
            isnew = atomicExch(stamp + w, tag) != tag;
          }
          const unsigned bal = __ballot_sync(FULL, isnew);
          if (isnew) queue[qlen + __popc(bal & lt)] = w;
          qlen += __popc(bal);
        }
      }
      __syncwarp();
      lv0 = start_len;
      lv1 = qlen;
    }
    const int q = qlen;
    if (q == 0) {
      if (lane == 0) jac[item] = 1.0;
      continue;
    }
    // ---- smallest ring h whose guaranteed radius holds >= q points
    const double2 pv = xy[v];
    const int cvx = cell_of(pv.x, gr.x0, gr.inv, gr.g), cvy = cell_of(pv.y, gr.y0, gr.inv, gr.g);
    // points of the square [cvx-h, cvx+h] x [cvy-h, cvy+h], rows of cells
    // being contiguous in the cell-sorted order
    auto for_square = [&](int h, auto&& fn) {
      const int x0 = max(cvx - h, 0), x1 = min(cvx + h, gr.g - 1);
      const int y0 = max(cvy - h, 0), y1 = min(cvy + h, gr.g - 1);
      for (int cy = y0; cy <= y1; cy++) {
        const long long a = cstart[(long long)cy * gr.g + x0];
        const long long b = cstart[(long long)cy * gr.g + x1 + 1];
        for (long long i = a + lane; i < b; i += 32) {
          const int w = __ldg(cpts + i);
          if (w != v) fn(w);
        }
      }
    };
    auto radius = [&](int h) -> double {
      // every point within (h-1) cells' distance lies inside the square
      // (cell indices round by at most one); the square covering the grid
      // holds every point
      if (h >= gr.g) return INFINITY;
      return (double)(h - 1) * gr.cell * (1.0 - 1e-9);
    };
    int h;
    {
      // start from the density estimate: q points need a disc of q / dens
      // cells (n points over g*g cells), radius h - 1
      const double dens = (double)n / ((double)gr.g * gr.g);
      h = 1 + (int)ceil(sqrt((double)q / dens / 3.14159265358979));
      if (h > gr.g) h = gr.g;
    }
    for (;;) {
      const double rad = radius(h);
      unsigned cnt = 0;
      for_square(h, [&](int w) { cnt += cdist_xy(pv, xy[w]) <= rad; });
      cnt = __reduce_add_sync(FULL, cnt);
      if (cnt >= (unsigned)q || h >= gr.g) break;
      h = h + (h + 1) / 2;
      if (h > gr.g) h = gr.g;
    }
    const double rad = radius(h);
    // ---- radix select of the rank-(q-1) key (dist bits, then id bits)
    unsigned long long dpre = 0;  // selected high bits of the distance key
    int rank = q - 1;             // 0-based rank within the current prefix class
    for (int pass = 0; pass < 8; pass++) {
      for (int i = lane; i < 256; i += 32) hh[i] = 0;
      __syncwarp();
      const int shift = 56 - 8 * pass;
      const unsigned long long dmask = pass == 0 ? 0ull : ~0ull << (64 - 8 * pass);
      for_square(h, [&](int w) {
        const double d = cdist_xy(pv, xy[w]);
        if (!(d <= rad)) return;
        const unsigned long long k = dkey(d);
        if ((k & dmask) != (dpre & dmask)) return;
        atomicAdd(&hh[(k >> shift) & 255], 1u);
      });
      __syncwarp();
      // digit where the cumulative count passes rank
      unsigned c8[8];
      unsigned tot = 0;
#pragma unroll
      for (int j = 0; j < 8; j++) {
        c8[j] = hh[lane * 8 + j];
        tot += c8[j];
      }
      unsigned incl = tot;
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
      }
      const unsigned excl = incl - tot;
      const bool here = excl <= (unsigned)rank && (unsigned)rank < incl;
      const unsigned hb = __ballot_sync(FULL, here);
      const int src = __ffs(hb) - 1;
      int digit = 0, below = 0;
      if (lane == src) {
        unsigned acc = excl;
        int j = 0;
        while (acc + c8[j] <= (unsigned)rank) {
          acc += c8[j];
          j++;
        }
        digit = lane * 8 + j;
        below = (int)acc;
      }
      digit = __shfl_sync(FULL, digit, src);
      below = __shfl_sync(FULL, below, src);
      rank -= below;
      dpre |= (unsigned long long)digit << shift;
      __syncwarp();
    }
    // dpre is the exact threshold distance D*; among points at exactly D*,
    // the rank-th smallest id is the threshold id W*
    const double dstar = __longlong_as_double((long long)dpre);
    unsigned wpre = 0;
    for (int pass = 0; pass < 4; pass++) {
      for (int i = lane; i < 256; i += 32) hh[i] = 0;
      __syncwarp();
      const int shift = 24 - 8 * pass;
      const unsigned wmask = pass == 0 ? 0u : ~0u << (32 - 8 * pass);
      for_square(h, [&](int w) {
        const double d = cdist_xy(pv, xy[w]);
        if (d != dstar) return;
        if (((unsigned)w & wmask) != (wpre & wmask)) return;
        atomicAdd(&hh[((unsigned)w >> shift) & 255], 1u);
      });
      __syncwarp();
      unsigned c8[8];
      unsigned tot = 0;
#pragma unroll
      for (int j = 0; j < 8; j++) {
        c8[j] = hh[lane * 8 + j];
        tot += c8[j];
      }
      unsigned incl = tot;
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
      }
      const unsigned excl = incl - tot;
      const bool here = excl <= (unsigned)rank && (unsigned)rank < incl;
      const unsigned hb = __ballot_sync(FULL, here);
      const int src = __ffs(hb) - 1;
      int digit = 0, below = 0;
      if (lane == src) {
        unsigned acc = excl;
        int j = 0;
        while (acc + c8[j] <= (unsigned)rank) {
          acc += c8[j];
          j++;
        }
        digit = lane * 8 + j;
        below = (int)acc;
      }
      digit = __shfl_sync(FULL, digit, src);
      below = __shfl_sync(FULL, below, src);
      rank -= below;
      wpre |= (unsigned)digit << shift;
      __syncwarp();
    }
    // ---- inter = hood members with (dist, id) <= (D*, W*)
    unsigned inter = 0;
    for (int i = lane; i < q; i += 32) {
      const int u = queue[i];
      const double d = cdist_xy(pv, xy[u]);
      inter += (d < dstar) || (d == dstar && (unsigned)u <= wpre);
    }
    inter = __reduce_add_sync(FULL, inter);
    if (lane == 0) jac[item] = (double)inter / (double)(2 * q - (int)inter);
    __syncwarp();
  }
}

__global__ void sum_doubles(const double* __restrict__ x, long long n, double* __restrict__ out) {
  __shared__ double sh[1024 / 32];
  double a = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) a += x[i];
  const double s = block_sum(a, sh);
  if (threadIdx.x == 0) *out = s;
}

struct NpWs {
  Grid* grid;
  int* cell;
  int* ids;
  int* cell_sorted;
  int* pts;
  long long* cstart;
  int* stamps;
  int* queues;
  double* jac;
  void* tmp;
  size_t tmp_bytes;
};

size_t np_layout(long long n, int g, int slots, char* base, NpWs* ws) {
  const long long ncell = (long long)g * g;
  size_t sort_b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sort_b, (const int*)nullptr, (int*)nullptr,
                                  (const int*)nullptr, (int*)nullptr, (int)(n > 0 ? n : 1));
  Carve c{base};
  NpWs w;
  w.grid = c.take<Grid>(1);
  w.cell = c.take<int>((size_t)n);
  w.ids = c.take<int>((size_t)n);
  w.cell_sorted = c.take<int>((size_t)n);
  w.pts = c.take<int>((size_t)n);
  w.cstart = c.take<long long>((size_t)ncell + 1);
  w.stamps = c.take<int>((size_t)n * (size_t)slots);
  w.queues = c.take<int>((size_t)n * (size_t)slots);
  w.jac = c.take<double>((size_t)n);
  w.tmp_bytes = sort_b;
  w.tmp = c.take<char>(sort_b);
  if (ws) *ws = w;
  return c.off;
}

int np_grid_side(long long n) {
  long long g = 1;
  while (g * g * 2 < n) g++;
  return (int)g;
}

}  // namespace
}  // namespace gu

using namespace gu;

// ------------------------------------------------------------------ stress
extern "C" size_t gu_stress_workspace_size(int64_t n) { return stress_layout(n, nullptr, nullptr); }

extern "C" int gu_stress(int64_t n, const int32_t* indptr, const int32_t* indices,
                         const double* coords_xy, int32_t rescale, const int32_t* sources,
                         int64_t nsources, double* out3, void* workspace, size_t ws_bytes,
                         void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 2 || n >= INT_MAX || (sources && (nsources < 1 || nsources > n))) {
    set_error("gu_stress: n=%lld nsources=%lld out of range (n < 2 is answered by the caller)",
              (long long)n, (long long)nsources);
    return GU_ERR_ARG;
  }
  StressWs ws;
  const size_t need = stress_layout(n, (char*)workspace, &ws);
  if (!workspace || ws_bytes < need) {
    set_error("gu_stress: workspace %zu < %zu", ws_bytes, need);
    return GU_ERR_WORKSPACE;
  }
  GU_CHECK(cudaMemsetAsync(ws.flag, 0, sizeof(int), st));
  GU_CHECK(cudaMemsetAsync(ws.sums, 0, 2 * sizeof(double2), st));
  GU_CHECK(cudaMemsetAsync(ws.acc, 0, sizeof(double2) * ST_CTAS, st));
  if (!rescale) {  // scale = 1 before the only pass
    stress_scale<<<1, 1, 0, st>>>(ws.sums, 0, ws.scale);
    GU_CHECK_LAUNCH("stress_scale");
  }
  for (int pass = rescale ? 0 : 1; pass < 2; pass++) {
    const int rc = stress_bfs_pass(n, indptr, indices, coords_xy, pass, ws.scale, ws.acc, ws.flag,
                                   ws.bfs, ws.bfs_bytes, ST_CTAS, sources, nsources, st);
    if (rc != GU_OK) return rc;
    reduce_acc<<<1, ST_THREADS, 0, st>>>(ws.acc, ST_CTAS, ws.sums + pass);
    GU_CHECK_LAUNCH("reduce_acc");
    if (pass == 0) {
      stress_scale<<<1, 1, 0, st>>>(ws.sums, rescale, ws.scale);
      GU_CHECK_LAUNCH("stress_scale");
    }
  }
  stress_finish<<<1, 1, 0, st>>>(ws.sums, ws.scale, ws.flag, out3);
  GU_CHECK_LAUNCH("stress_finish");
  return GU_OK;
}

// --------------------------------------------------------------- crossings
extern "C" int gu_crossings_grid(int64_t n, const double* coords_xy, int32_t g, void* grid_out,
                                 void* stream) {
  if (g < 1) {
    set_error("gu_crossings_grid: g=%d", g);
    return GU_ERR_ARG;
  }
  grid_from_bbox<<<1, 1024, 0, (cudaStream_t)stream>>>((const double2*)coords_xy, n, g,
                                                       (Grid*)grid_out);
  GU_CHECK_LAUNCH("grid_from_bbox");
  return GU_OK;
}

extern "C" size_t gu_grid_bytes(void) { return sizeof(Grid); }

extern "C" int gu_crossings_incidences(int64_t m, const int32_t* edges, const double* coords_xy,
                                       const void* grid, int64_t* out_counts, void* stream) {
  if (m < 0) {
    set_error("gu_crossings_incidences: m=%lld", (long long)m);
    return GU_ERR_ARG;
  }
  if (m == 0) return GU_OK;
  cross_raster<false><<<148 * 8, 256, 0, (cudaStream_t)stream>>>(
      m, (const int2*)edges, (const double2*)coords_xy, (const Grid*)grid, (long long*)out_counts,
      nullptr, nullptr, nullptr);
  GU_CHECK_LAUNCH("cross_raster(count)");
  return GU_OK;
}

extern "C" size_t gu_crossings_workspace_size(int64_t m, int64_t n_inc, int32_t g) {
  return cross_layout(m, n_inc, g, nullptr, nullptr);
}

// edges: int32 (m, 2); grid from gu_crossings_grid (same g); n_inc = the sum
// of gu_crossings_incidences; out_count: device uint64
extern "C" int gu_crossings(int64_t m, const int32_t* edges, const double* coords_xy,
                            const void* grid, int32_t g, int64_t n_inc, uint64_t* out_count,
                            void* workspace, size_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (m < 0 || g < 1 || n_inc < 0 || n_inc >= INT_MAX) {
    set_error("gu_crossings: bad arguments (m=%lld g=%d incidences=%lld)", (long long)m, g,
              (long long)n_inc);
    return GU_ERR_ARG;
  }
  CrossWs ws;
  const size_t need = cross_layout(m, n_inc, g, (char*)workspace, &ws);
  if (!workspace || ws_bytes < need) {
    set_error("gu_crossings: workspace %zu < %zu", ws_bytes, need);
    return GU_ERR_WORKSPACE;
  }
  GU_CHECK(cudaMemsetAsync(out_count, 0, sizeof(uint64_t), st));
  if (m < 2 || n_inc == 0) return GU_OK;
  const long long ncell = (long long)g * g;
  const Grid* gr = (const Grid*)grid;
  cross_raster<false><<<148 * 8, 256, 0, st>>>(m, (const int2*)edges, (const double2*)coords_xy,
                                                gr, ws.ecount, nullptr, nullptr, nullptr);
  GU_CHECK_LAUNCH("cross_raster(count)");
  GU_CHECK(cudaMemsetAsync(ws.ecount + m, 0, sizeof(long long), st));
  size_t tb = ws.tmp_bytes;
  GU_CHECK(cub::DeviceScan::ExclusiveSum(ws.tmp, tb, ws.ecount, ws.eoff, (int)(m + 1), st));
  cross_raster<true><<<148 * 8, 256, 0, st>>>(m, (const int2*)edges, (const double2*)coords_xy, gr,
                                               nullptr, ws.eoff, ws.inc_cell, ws.inc_edge);
  GU_CHECK_LAUNCH("cross_raster(fill)");
  int end_bit = 1;
  while (end_bit < 31 && (1ll << end_bit) < ncell) end_bit++;
  tb = ws.tmp_bytes;
  GU_CHECK(cub::DeviceRadixSort::SortPairs(ws.tmp, tb, ws.inc_cell, ws.sorted_cell, ws.inc_edge,
                                           ws.sorted_edge, (int)n_inc, 0, end_bit, st));
  cell_starts<<<148 * 8, 256, 0, st>>>(ncell, ws.sorted_cell, n_inc, ws.cstart);
  GU_CHECK_LAUNCH("cell_starts");
  cell_pair_counts<<<148 * 8, 256, 0, st>>>(ncell, ws.cstart, ws.pstart);
  GU_CHECK_LAUNCH("cell_pair_counts");
  GU_CHECK(cudaMemsetAsync(ws.pstart + ncell, 0, sizeof(long long), st));
  tb = ws.tmp_bytes;
  GU_CHECK(cub::DeviceScan::ExclusiveSum(ws.tmp, tb, ws.pstart, ws.pstart, (int)(ncell + 1), st));
  cross_pairs<<<148 * 16, 256, 0, st>>>(ncell, ws.pstart, ws.cstart, ws.sorted_edge,
                                        (const int2*)edges, (const double2*)coords_xy, gr,
                                        (unsigned long long*)out_count);
  GU_CHECK_LAUNCH("cross_pairs");
  return GU_OK;
}

// ----------------------------------------------------- neighborhood pres.
extern "C" size_t gu_np_workspace_size(int64_t n, int32_t slots) {
  return np_layout(n, np_grid_side(n), slots > 0 ? slots : 1, nullptr, nullptr);
}

// out_sum: device double = sum of the Jaccard terms over every vertex, or
// over the nsources distinct vertices in `sources` (sampled estimator) when
// it is non-null; the caller divides.  slots: concurrent warps, each with 2n
// ints of scratch
extern "C" int gu_neighborhood_preservation(int64_t n, const int32_t* indptr,
                                            const int32_t* indices, const double* coords_xy,
                                            int32_t r, int32_t slots, const int32_t* sources,
                                            int64_t nsources, double* out_sum, void* workspace,
                                            size_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 1 || n >= INT_MAX || (sources && (nsources < 1 || nsources > n))) {
    set_error("gu_neighborhood_preservation: n=%lld nsources=%lld", (long long)n,
              (long long)nsources);
    return GU_ERR_ARG;
  }
  if (slots < 1) slots = 1;
  if (r < 1) r = 1;  // metrics.py:55-58: r <= 1 is the adjacency itself
  const int g = np_grid_side(n);
  NpWs ws;
  const size_t need = np_layout(n, g, slots, (char*)workspace, &ws);
  if (!workspace || ws_bytes < need) {
    set_error("gu_neighborhood_preservation: workspace %zu < %zu", ws_bytes, need);
    return GU_ERR_WORKSPACE;
  }
  const double2* xy = (const double2*)coords_xy;
  grid_from_bbox<<<1, 1024, 0, st>>>(xy, n, g, ws.grid);
  GU_CHECK_LAUNCH("grid_from_bbox");
  np_cells<<<148 * 8, 256, 0, st>>>(xy, (int)n, ws.grid, ws.cell, ws.ids);
  GU_CHECK_LAUNCH("np_cells");
  const long long ncell = (long long)g * g;
  int end_bit = 1;
  while (end_bit < 31 && (1ll << end_bit) < ncell) end_bit++;
  size_t tb = ws.tmp_bytes;
  GU_CHECK(cub::DeviceRadixSort::SortPairs(ws.tmp, tb, ws.cell, ws.cell_sorted, ws.ids, ws.pts,
                                           (int)n, 0, end_bit, st));
  cell_starts<<<148 * 8, 256, 0, st>>>(ncell, ws.cell_sorted, n, ws.cstart);
  GU_CHECK_LAUNCH("cell_starts");
  GU_CHECK(cudaMemsetAsync(ws.stamps, 0, sizeof(int) * (size_t)n * (size_t)slots, st));
  const unsigned blocks = (unsigned)((slots + NP_WARPS - 1) / NP_WARPS);
  const int nitems = sources ? (int)nsources : (int)n;
  np_kernel<<<blocks, NP_WARPS * 32, 0, st>>>((int)n, indptr, indices, xy, r, ws.grid, ws.cstart,
                                              ws.pts, ws.stamps, ws.queues, slots, sources, nitems,
                                              ws.jac);
  GU_CHECK_LAUNCH("np_kernel");
  sum_doubles<<<1, 1024, 0, st>>>(ws.jac, nitems, out_sum);
  GU_CHECK_LAUNCH("sum_doubles");
  return GU_OK;
}
