// sparsify.cu -- effective resistances and the n log2 n spectral sparsifier
// (/root/reference/pkg/src/graph_umap/sparsify.py).
//
//   effective_resistance_exact   sparsify.py:49-84   r_e from the grounded
//       Laplacian inverse X (dense, n <= cap; the inverse itself is a cuSOLVER
//       Cholesky in the host wrapper): r = X_uu + X_vv - 2 X_uv (X_0* = 0)
//   effective_resistance_approx  sparsify.py:87-143  q Rademacher projections
//       of the incidence matrix, q Jacobi-PCG Laplacian solves (block PCG over
//       a row-major n x q matrix), r_e = sum_i (y_i[u] - y_i[v])^2.  The signs
//       are counter-based (hash of seed, i, edge) instead of numpy's stream.
//   sparsify                     sparsify.py:176-205 lexsort by (-r, u, v),
//       maximum spanning tree (Boruvka under the strict sort-position order
//       = Kruskal's tree), then the budget in sort order.
#include <climits>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "common.cuh"
#include "gumap.h"

namespace gu {
namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// --------------------------------------------------------------- exact
__global__ void sp_exact_gather(long long m, const int2* __restrict__ edges,
                                const double* __restrict__ X, int nm1, double* __restrict__ r) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += (long long)gridDim.x * blockDim.x) {
    const int u = edges[e].x, v = edges[e].y;  // grounded at vertex 0
    const double xuu = u > 0 ? X[(long long)(u - 1) * nm1 + (u - 1)] : 0.0;
    const double xvv = v > 0 ? X[(long long)(v - 1) * nm1 + (v - 1)] : 0.0;
    const double xuv = (u > 0 && v > 0) ? X[(long long)(u - 1) * nm1 + (v - 1)] : 0.0;
    r[e] = (xuu - xuv) - (xuv - xvv);  // phi_u - phi_v for b = e_u - e_v
  }
}

// ------------------------------------------------------------- sketch
// B[v][i] = sum over edges (a < b) at v of sign_i(a, b) * (+1 at a, -1 at b) / sqrt(q)
__global__ void sp_project(int n, int q, const int* __restrict__ indptr,
                           const int* __restrict__ indices, unsigned long long seed, double scale,
                           double* __restrict__ B) {
  const long long total = (long long)n * q;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int v = (int)(t / q), i = (int)(t - (long long)v * q);
    const int b = __ldg(indptr + v), e = __ldg(indptr + v + 1);
    double s = 0.0;
    for (int p = b; p < e; p++) {
      const int u = __ldg(indices + p);
      const unsigned lo = (unsigned)min(u, v), hi = (unsigned)max(u, v);
      const unsigned long long h =
          mix64(seed ^ mix64(((unsigned long long)i << 32) ^ 0x5851F42D4C957F2DULL) ^
                (((unsigned long long)lo << 32) | hi));
      const double sg = (h >> 63) ? 1.0 : -1.0;
      s += v < u ? sg : -sg;
    }
    B[t] = s * scale;
  }
}

// Y_out = L Y  (row-major n x q; L = D - A); one warp per row, lanes over q
__global__ void sp_lap_spmm(int n, int q, const int* __restrict__ indptr,
                            const int* __restrict__ indices, const double* __restrict__ Y,
                            double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (int v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n;
       v += (gridDim.x * blockDim.x) >> 5) {
    const int b = __ldg(indptr + v), e = __ldg(indptr + v + 1);
    const double d = (double)(e - b);
    for (int c = lane; c < q; c += 32) {
      double s = d * Y[(long long)v * q + c];
      for (int p = b; p < e; p++) s -= Y[(long long)__ldg(indices + p) * q + c];
      out[(long long)v * q + c] = s;
    }
  }
}

// partial[blk][c] = sum over this block's rows of A[r][c] * B[r][c]
__global__ void sp_coldot_partial(int n, int q, const double* __restrict__ A,
                                  const double* __restrict__ Bm, double* __restrict__ partial) {
  // thread t owns columns t, t + blockDim.x, ... ; rows strided over blocks
  for (int c = threadIdx.x; c < q; c += blockDim.x) {
    double s = 0.0;
    for (int r = blockIdx.x; r < n; r += gridDim.x) s += A[(long long)r * q + c] * Bm[(long long)r * q + c];
    partial[(long long)blockIdx.x * q + c] = s;
  }
}

__global__ void sp_coldot_final(int q, int nblk, const double* __restrict__ partial,
                                double* __restrict__ out) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < q; c += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nblk; b++) s += partial[(long long)b * q + c];
    out[c] = s;
  }
}

// PCG state per column: rz, alpha/beta, ||b||, converged flag
struct ColState {
  double rz, bnorm, pap, rr;
  int done;
};

__global__ void sp_cg_init_cols(int q, const double* __restrict__ rz, const double* __restrict__ bb,
                                ColState* __restrict__ st, double rtol, int* __restrict__ active) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < q; c += gridDim.x * blockDim.x) {
    st[c].rz = rz[c];
    st[c].bnorm = sqrt(bb[c]);
    st[c].done = (sqrt(bb[c]) == 0.0) ? 1 : 0;
    if (!st[c].done) atomicAdd(active, 1);
  }
}

// Y += a P ; R -= a AP ; Z = R / d   (a = rz / pAp for live columns)
__global__ void sp_cg_step1(int n, int q, const int* __restrict__ indptr,
                            const double* __restrict__ pap, const ColState* __restrict__ st,
                            double* __restrict__ Y, double* __restrict__ R,
                            const double* __restrict__ P, const double* __restrict__ AP,
                            double* __restrict__ Z) {
  const long long total = (long long)n * q;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int v = (int)(t / q), c = (int)(t - (long long)v * q);
    if (st[c].done) continue;
    const double a = st[c].rz / pap[c];
    Y[t] += a * P[t];
    R[t] -= a * AP[t];
    Z[t] = R[t] / (double)(indptr[v + 1] - indptr[v]);
  }
}

// convergence (||r|| <= rtol ||b||, scipy cg's test) and beta
__global__ void sp_cg_cols(int q, const double* __restrict__ rz_new, const double* __restrict__ rr,
                           ColState* __restrict__ st, double rtol, double* __restrict__ beta,
                           int* __restrict__ active) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < q; c += gridDim.x * blockDim.x) {
    if (st[c].done) {
      beta[c] = 0.0;
      continue;
    }
    st[c].rr = rr[c];
    if (sqrt(rr[c]) <= rtol * st[c].bnorm) {
      st[c].done = 1;
      beta[c] = 0.0;
      continue;
    }
    atomicAdd(active, 1);
    beta[c] = rz_new[c] / st[c].rz;
    st[c].rz = rz_new[c];
  }
}

// Z = R / d (Jacobi)
__global__ void sp_jacobi(int n, int q, const int* __restrict__ indptr, const double* __restrict__ R,
                          double* __restrict__ Z) {
  const long long total = (long long)n * q;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int v = (int)(t / q);
    Z[t] = R[t] / (double)(indptr[v + 1] - indptr[v]);
  }
}

// P = Z + beta P
__global__ void sp_cg_step2(int n, int q, const double* __restrict__ beta,
                            const ColState* __restrict__ st, const double* __restrict__ Z,
                            double* __restrict__ P) {
  const long long total = (long long)n * q;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(t % q);
    if (st[c].done) continue;
    P[t] = Z[t] + beta[c] * P[t];
  }
}

// acc[e] = sum_i (Y[u][i] - Y[v][i])^2 ; one warp per edge
__global__ void sp_edge_acc(long long m, int q, const int2* __restrict__ edges,
                            const double* __restrict__ Y, double* __restrict__ acc) {
  const int lane = threadIdx.x & 31;
  for (long long e = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < m;
       e += ((long long)gridDim.x * blockDim.x) >> 5) {
    const int u = edges[e].x, v = edges[e].y;
    double s = 0.0;
    for (int c = lane; c < q; c += 32) {
      const double d = Y[(long long)u * q + c] - Y[(long long)v * q + c];
      s += d * d;
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(FULL, s, o);
    if (lane == 0) acc[e] = s;
  }
}

// ---------------------------------------------------------- selection
// descending r, stable in edge id: key = ~bits(r) (r >= 0)
__global__ void sp_sort_keys(long long m, const double* __restrict__ r,
                             unsigned long long* __restrict__ key, int* __restrict__ id) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += (long long)gridDim.x * blockDim.x) {
    double x = r[e];
    if (x == 0.0) x = 0.0;  // -0.0 -> +0.0
    key[e] = ~(unsigned long long)__double_as_longlong(x);
    id[e] = (int)e;
  }
}

__device__ __forceinline__ int uf_find(int* parent, int x) {
  int p = parent[x];
  while (p != x) {
    const int gp = parent[p];
    if (gp != p) parent[x] = gp;
    x = p;
    p = gp;
  }
  return x;
}

__global__ void sp_iota(int n, int* __restrict__ a) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = i;
}

__global__ void sp_fill(int n, int* __restrict__ a, int v) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = v;
}

// Boruvka round, step 1: every root takes its best (lowest sort position)
// incident edge to another component
__global__ void sp_bv_best(long long m, const int2* __restrict__ sorted_edges, int* parent,
                           int* __restrict__ best) {
  for (long long pos = (long long)blockIdx.x * blockDim.x + threadIdx.x; pos < m;
       pos += (long long)gridDim.x * blockDim.x) {
    const int2 e = sorted_edges[pos];
    const int ru = uf_find(parent, e.x), rv = uf_find(parent, e.y);
    if (ru == rv) continue;
    atomicMin(best + ru, (int)pos);
    atomicMin(best + rv, (int)pos);
  }
}

// step 2: mark the chosen edges, then hook their endpoints' components
__global__ void sp_bv_mark(int n, const int* __restrict__ best, unsigned char* __restrict__ in_tree,
                           int* __restrict__ progress) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const int b = best[v];
    if (b != INT_MAX) {
      in_tree[b] = 1;
      *progress = 1;
    }
  }
}

__global__ void sp_bv_hook(int n, const int* __restrict__ best, const int2* __restrict__ sorted_edges,
                           int* parent) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const int b = best[v];
    if (b == INT_MAX) continue;
    const int2 e = sorted_edges[b];
    for (;;) {
      int ru = uf_find(parent, e.x), rv = uf_find(parent, e.y);
      if (ru == rv) break;
      if (ru < rv) {
        const int t = ru;
        ru = rv;
        rv = t;
      }
      if (atomicCAS(parent + ru, ru, rv) == ru) break;
    }
  }
}

__global__ void sp_gather_edges(long long m, const int* __restrict__ order, const int2* __restrict__ edges,
                                int2* __restrict__ sorted_edges) {
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < m;
       p += (long long)gridDim.x * blockDim.x)
    sorted_edges[p] = edges[order[p]];
}

__global__ void sp_nontree(long long m, const unsigned char* __restrict__ in_tree,
                           int* __restrict__ flag) {
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < m;
       p += (long long)gridDim.x * blockDim.x)
    flag[p] = in_tree[p] ? 0 : 1;
}

// keep tree edges and the first `budget` non-tree edges in sort order
__global__ void sp_keep(long long m, const unsigned char* __restrict__ in_tree,
                        const int* __restrict__ nt_before, long long budget,
                        const int* __restrict__ order, unsigned char* __restrict__ keep_by_id) {
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < m;
       p += (long long)gridDim.x * blockDim.x)
    keep_by_id[order[p]] = (in_tree[p] || (long long)nt_before[p] < budget) ? 1 : 0;
}

constexpr int SP_THREADS = 256;
constexpr int SP_BLOCKS = 148 * 8;
constexpr int SP_DOT_BLOCKS = 148 * 4;

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

struct SketchWs {
  double *B, *Y, *R, *Z, *P, *AP, *partial, *d1, *d2, *beta;
  ColState* st;
  int* active;
};

size_t sketch_layout(long long n, int q, char* base, SketchWs* ws) {
  Carve c{base};
  SketchWs w;
  const size_t nq = (size_t)n * (size_t)q;
  w.B = c.take<double>(nq);
  w.Y = c.take<double>(nq);
  w.R = c.take<double>(nq);
  w.Z = c.take<double>(nq);
  w.P = c.take<double>(nq);
  w.AP = c.take<double>(nq);
  w.partial = c.take<double>((size_t)SP_DOT_BLOCKS * q);
  w.d1 = c.take<double>(q);
  w.d2 = c.take<double>(q);
  w.beta = c.take<double>(q);
  w.st = c.take<ColState>(q);
  w.active = c.take<int>(1);
  if (ws) *ws = w;
  return c.off;
}

int coldot(int n, int q, const double* A, const double* B, double* partial, double* out,
           cudaStream_t st) {
  sp_coldot_partial<<<SP_DOT_BLOCKS, SP_THREADS, 0, st>>>(n, q, A, B, partial);
  GU_CHECK_LAUNCH("sp_coldot_partial");
  sp_coldot_final<<<(q + 255) / 256, 256, 0, st>>>(q, SP_DOT_BLOCKS, partial, out);
  GU_CHECK_LAUNCH("sp_coldot_final");
  return GU_OK;
}

struct SelWs {
  unsigned long long *k0, *k1;
  int *id0, *order;
  int2* sorted_edges;
  int* parent;
  int* best;
  unsigned char* in_tree;
  int* nt;
  int* nt_before;
  int* progress;
  void* tmp;
  size_t tmp_bytes;
};

size_t sel_layout(long long n, long long m, char* base, SelWs* ws) {
  size_t sb = 0, cb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sb, (const unsigned long long*)nullptr,
                                  (unsigned long long*)nullptr, (const int*)nullptr, (int*)nullptr,
                                  (int)(m > 0 ? m : 1));
  cub::DeviceScan::ExclusiveSum(nullptr, cb, (const int*)nullptr, (int*)nullptr,
                                (int)(m > 0 ? m : 1));
  Carve c{base};
  SelWs w;
  w.k0 = c.take<unsigned long long>((size_t)m);
  w.k1 = c.take<unsigned long long>((size_t)m);
  w.id0 = c.take<int>((size_t)m);
  w.order = c.take<int>((size_t)m);
  w.sorted_edges = c.take<int2>((size_t)m);
  w.parent = c.take<int>((size_t)n);
  w.best = c.take<int>((size_t)n);
  w.in_tree = c.take<unsigned char>((size_t)m);
  w.nt = c.take<int>((size_t)m);
  w.nt_before = c.take<int>((size_t)m);
  w.progress = c.take<int>(1);
  w.tmp_bytes = sb > cb ? sb : cb;
  w.tmp = c.take<char>(w.tmp_bytes);
  if (ws) *ws = w;
  return c.off;
}

}  // namespace
}  // namespace gu

using namespace gu;

extern "C" int gu_resistance_exact_gather(int64_t m, const int32_t* edges, const double* X,
                                          int64_t n, double* out_r, void* stream) {
  if (m < 0 || n < 1 || n >= INT_MAX) {
    set_error("gu_resistance_exact_gather: bad arguments");
    return GU_ERR_ARG;
  }
  if (m == 0) return GU_OK;
  sp_exact_gather<<<SP_BLOCKS, SP_THREADS, 0, (cudaStream_t)stream>>>(
      m, (const int2*)edges, X, (int)(n - 1), out_r);
  GU_CHECK_LAUNCH("sp_exact_gather");
  return GU_OK;
}

extern "C" size_t gu_resistance_sketch_workspace_size(int64_t n, int32_t q) {
  return sketch_layout(n, q, nullptr, nullptr);
}

// out_r[e] = sum over q projections of (y_i[u] - y_i[v])^2 ; host_iters
// (host int): PCG iterations run; returns GU_ERR_UNSUPPORTED (not converged)
// with out_resid (host double) = the worst column residual when maxiter is hit
extern "C" int gu_resistance_sketch(int64_t n, const int32_t* indptr, const int32_t* indices,
                                    int64_t m, const int32_t* edges, int32_t q, uint64_t seed,
                                    double rtol, int32_t maxiter, double* out_r, int32_t* host_iters,
                                    double* host_resid, void* workspace, size_t ws_bytes,
                                    void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 1 || n >= INT_MAX || q < 1 || m < 0) {
    set_error("gu_resistance_sketch: bad arguments");
    return GU_ERR_ARG;
  }
  SketchWs ws;
  const size_t need = sketch_layout(n, q, (char*)workspace, &ws);
  if (!workspace || ws_bytes < need) {
    set_error("gu_resistance_sketch: workspace %zu < %zu", ws_bytes, need);
    return GU_ERR_WORKSPACE;
  }
  const int N = (int)n;
  const size_t nq = (size_t)n * q;
  sp_project<<<SP_BLOCKS, SP_THREADS, 0, st>>>(N, q, indptr, indices, seed, 1.0 / sqrt((double)q), ws.B);
  GU_CHECK_LAUNCH("sp_project");
  // x0 = 0: R = B, Z = D^-1 R, P = Z (scipy cg's first iteration)
  GU_CHECK(cudaMemsetAsync(ws.Y, 0, sizeof(double) * nq, st));
  GU_CHECK(cudaMemcpyAsync(ws.R, ws.B, sizeof(double) * nq, cudaMemcpyDeviceToDevice, st));
  int rc = coldot(N, q, ws.B, ws.B, ws.partial, ws.d2, st);  // ||b||^2
  if (rc != GU_OK) return rc;
  sp_jacobi<<<SP_BLOCKS, SP_THREADS, 0, st>>>(N, q, indptr, ws.R, ws.Z);
  GU_CHECK_LAUNCH("sp_jacobi");
  GU_CHECK(cudaMemcpyAsync(ws.P, ws.Z, sizeof(double) * nq, cudaMemcpyDeviceToDevice, st));
  rc = coldot(N, q, ws.R, ws.Z, ws.partial, ws.d1, st);  // rz
  if (rc != GU_OK) return rc;
  GU_CHECK(cudaMemsetAsync(ws.active, 0, sizeof(int), st));
  GU_CHECK(cudaMemsetAsync(ws.st, 0, sizeof(ColState) * q, st));
  sp_cg_init_cols<<<(q + 255) / 256, 256, 0, st>>>(q, ws.d1, ws.d2, ws.st, rtol, ws.active);
  GU_CHECK_LAUNCH("sp_cg_init_cols");
  int it = 0, active = 1;
  for (it = 0; it < maxiter; it++) {
    sp_lap_spmm<<<SP_BLOCKS, SP_THREADS, 0, st>>>(N, q, indptr, indices, ws.P, ws.AP);
    GU_CHECK_LAUNCH("sp_lap_spmm");
    rc = coldot(N, q, ws.P, ws.AP, ws.partial, ws.d1, st);  // pAp
    if (rc != GU_OK) return rc;
    sp_cg_step1<<<SP_BLOCKS, SP_THREADS, 0, st>>>(N, q, indptr, ws.d1, ws.st, ws.Y, ws.R, ws.P,
                                                  ws.AP, ws.Z);
    GU_CHECK_LAUNCH("sp_cg_step1");
    rc = coldot(N, q, ws.R, ws.Z, ws.partial, ws.d1, st);  // rz_new
    if (rc != GU_OK) return rc;
    rc = coldot(N, q, ws.R, ws.R, ws.partial, ws.d2, st);  // rr
    if (rc != GU_OK) return rc;
    GU_CHECK(cudaMemsetAsync(ws.active, 0, sizeof(int), st));
    sp_cg_cols<<<(q + 255) / 256, 256, 0, st>>>(q, ws.d1, ws.d2, ws.st, rtol, ws.beta, ws.active);
    GU_CHECK_LAUNCH("sp_cg_cols");
    sp_cg_step2<<<SP_BLOCKS, SP_THREADS, 0, st>>>(N, q, ws.beta, ws.st, ws.Z, ws.P);
    GU_CHECK_LAUNCH("sp_cg_step2");
    if ((it & 7) == 7) {
      GU_CHECK(cudaMemcpyAsync(&active, ws.active, sizeof(int), cudaMemcpyDeviceToHost, st));
      GU_CHECK(cudaStreamSynchronize(st));
      if (active == 0) {
        it++;
        break;
      }
    }
  }
  GU_CHECK(cudaMemcpyAsync(&active, ws.active, sizeof(int), cudaMemcpyDeviceToHost, st));
  GU_CHECK(cudaStreamSynchronize(st));
  *host_iters = it;
  if (active != 0) {
    std::vector<double> rr(q);
    GU_CHECK(cudaMemcpy(rr.data(), ws.d2, sizeof(double) * q, cudaMemcpyDeviceToHost));
    double worst = 0.0;
    for (double x : rr) worst = x > worst ? x : worst;
    *host_resid = sqrt(worst);
    set_error("CG did not converge within %d iterations (residual %.3e)", maxiter, *host_resid);
    return GU_ERR_UNSUPPORTED;
  }
  *host_resid = 0.0;
  sp_edge_acc<<<SP_BLOCKS, SP_THREADS, 0, st>>>(m, q, (const int2*)edges, ws.Y, out_r);
  GU_CHECK_LAUNCH("sp_edge_acc");
  return GU_OK;
}

extern "C" size_t gu_sparsify_workspace_size(int64_t n, int64_t m) {
  return sel_layout(n, m, nullptr, nullptr);
}

// keep (device uint8[m], by edge id): the max-resistance spanning tree plus
// the first (target - tree) non-tree edges in (-r, u, v) order
extern "C" int gu_sparsify_select(int64_t n, int64_t m, const int32_t* edges, const double* r,
                                  int64_t target, uint8_t* keep, int32_t* host_tree_edges,
                                  void* workspace, size_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 1 || n >= INT_MAX || m < 0 || m >= INT_MAX || target < 0) {
    set_error("gu_sparsify_select: bad arguments");
    return GU_ERR_ARG;
  }
  SelWs ws;
  const size_t need = sel_layout(n, m, (char*)workspace, &ws);
  if (!workspace || ws_bytes < need) {
    set_error("gu_sparsify_select: workspace %zu < %zu", ws_bytes, need);
    return GU_ERR_WORKSPACE;
  }
  if (m == 0) {
    *host_tree_edges = 0;
    return GU_OK;
  }
  const int M = (int)m, N = (int)n;
  sp_sort_keys<<<SP_BLOCKS, SP_THREADS, 0, st>>>(m, r, ws.k0, ws.id0);
  GU_CHECK_LAUNCH("sp_sort_keys");
  size_t tb = ws.tmp_bytes;
  GU_CHECK(cub::DeviceRadixSort::SortPairs(ws.tmp, tb, ws.k0, ws.k1, ws.id0, ws.order, M, 0, 64, st));
  sp_gather_edges<<<SP_BLOCKS, SP_THREADS, 0, st>>>(m, ws.order, (const int2*)edges, ws.sorted_edges);
  GU_CHECK_LAUNCH("sp_gather_edges");
  sp_iota<<<SP_BLOCKS, SP_THREADS, 0, st>>>(N, ws.parent);
  GU_CHECK_LAUNCH("sp_iota");
  GU_CHECK(cudaMemsetAsync(ws.in_tree, 0, (size_t)m, st));
  for (int round = 0; round < 64; round++) {
    sp_fill<<<SP_BLOCKS, SP_THREADS, 0, st>>>(N, ws.best, INT_MAX);
    GU_CHECK_LAUNCH("sp_fill");
    sp_bv_best<<<SP_BLOCKS, SP_THREADS, 0, st>>>(m, ws.sorted_edges, ws.parent, ws.best);
    GU_CHECK_LAUNCH("sp_bv_best");
    GU_CHECK(cudaMemsetAsync(ws.progress, 0, sizeof(int), st));
    sp_bv_mark<<<SP_BLOCKS, SP_THREADS, 0, st>>>(N, ws.best, ws.in_tree, ws.progress);
    GU_CHECK_LAUNCH("sp_bv_mark");
    sp_bv_hook<<<SP_BLOCKS, SP_THREADS, 0, st>>>(N, ws.best, ws.sorted_edges, ws.parent);
    GU_CHECK_LAUNCH("sp_bv_hook");
    int progress = 0;
    GU_CHECK(cudaMemcpyAsync(&progress, ws.progress, sizeof(int), cudaMemcpyDeviceToHost, st));
    GU_CHECK(cudaStreamSynchronize(st));
    if (!progress) break;
  }
  sp_nontree<<<SP_BLOCKS, SP_THREADS, 0, st>>>(m, ws.in_tree, ws.nt);
  GU_CHECK_LAUNCH("sp_nontree");
  tb = ws.tmp_bytes;
  GU_CHECK(cub::DeviceScan::ExclusiveSum(ws.tmp, tb, ws.nt, ws.nt_before, M, st));
  int last_nt = 0, last_before = 0;
  GU_CHECK(cudaMemcpyAsync(&last_nt, ws.nt + (m - 1), sizeof(int), cudaMemcpyDeviceToHost, st));
  GU_CHECK(cudaMemcpyAsync(&last_before, ws.nt_before + (m - 1), sizeof(int), cudaMemcpyDeviceToHost, st));
  GU_CHECK(cudaStreamSynchronize(st));
  const long long nontree = (long long)last_nt + last_before;
  const long long tree = m - nontree;
  long long budget = target - tree;
  if (budget < 0) budget = 0;
  *host_tree_edges = (int32_t)tree;
  sp_keep<<<SP_BLOCKS, SP_THREADS, 0, st>>>(m, ws.in_tree, ws.nt_before, budget, ws.order, keep);
  GU_CHECK_LAUNCH("sp_keep");
  return GU_OK;
}
