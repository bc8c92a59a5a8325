// spectral.cu -- the deflated normalized-Laplacian operator of spectral_init
// (/root/reference/pkg/src/graph_umap/layout.py:221-304).
//
// The reference runs ARPACK (eigsh, k=1, 'LM', ncv=32, tol=1e-6) on
//   y = P (x' + D^-1/2 A D^-1/2 x'),  x' = P x,  P = I - B B^T
// (layout.py:270-273; 2I - L_sym with the trivial and found eigenvectors B
// deflated).  This file is that operator: two deterministic dot products
// against B, a projection, and the SpMV with 8 lanes per row.  The restarted
// Lanczos around it lives in layout.spectral_init (dense 32-column algebra).
#include <climits>

#include "common.cuh"
#include "gumap.h"

namespace gu {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int SP_THREADS = 256;
constexpr int SP_DOT_BLOCKS = 148 * 4;
constexpr int SP_MAX_BASIS = 4;

__global__ void spec_degree(int n, const int* __restrict__ indptr, double* __restrict__ inv_sqrt,
                            double* __restrict__ sqrt_deg) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const double d = (double)(indptr[v + 1] - indptr[v]);
    const double r = sqrt(d);
    inv_sqrt[v] = 1.0 / r;  // layout.py:212 (isolated vertices excluded by the caller)
    sqrt_deg[v] = r;
  }
}

// partial[j][block] = sum over this block's rows of B_j[i] * x[i]
__global__ void __launch_bounds__(SP_THREADS)
    spec_dots_partial(int n, const double* __restrict__ B, int nb, const double* __restrict__ x,
                      double* __restrict__ partial) {
  __shared__ double sh[SP_MAX_BASIS][SP_THREADS / 32];
  double acc[SP_MAX_BASIS] = {0.0, 0.0, 0.0, 0.0};
  for (int i = blockIdx.x * SP_THREADS + threadIdx.x; i < n; i += gridDim.x * SP_THREADS) {
    const double xi = x[i];
#pragma unroll
    for (int j = 0; j < SP_MAX_BASIS; j++)
      if (j < nb) acc[j] = fma(B[(long long)j * n + i], xi, acc[j]);
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < SP_MAX_BASIS; j++) {
    double v = acc[j];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(FULL, v, o);
    if (lane == 0) sh[j][w] = v;
  }
  __syncthreads();
  if (threadIdx.x < nb) {
    double s = 0.0;
    for (int k = 0; k < SP_THREADS / 32; k++) s += sh[threadIdx.x][k];
    partial[threadIdx.x * gridDim.x + blockIdx.x] = s;
  }
}

// coef[j] = sum of partial[j][*] in a fixed order
__global__ void spec_dots_final(const double* __restrict__ partial, int nb, int nblocks,
                                double* __restrict__ coef) {
  __shared__ double sh[SP_THREADS / 32];
  for (int j = 0; j < nb; j++) {
    double v = 0.0;
    for (int k = threadIdx.x; k < nblocks; k += blockDim.x) v += partial[j * nblocks + k];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(FULL, v, o);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) sh[w] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int k = 0; k < (int)(blockDim.x >> 5); k++) s += sh[k];
      coef[j] = s;
    }
    __syncthreads();
  }
}

// out = x - B coef ; if z: z = inv_sqrt * out
__global__ void spec_project(int n, const double* __restrict__ B, int nb,
                             const double* __restrict__ coef, const double* __restrict__ x,
                             double* __restrict__ out, const double* __restrict__ inv_sqrt,
                             double* __restrict__ z) {
  double c[SP_MAX_BASIS];
#pragma unroll
  for (int j = 0; j < SP_MAX_BASIS; j++) c[j] = j < nb ? coef[j] : 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double v = x[i];
#pragma unroll
    for (int j = 0; j < SP_MAX_BASIS; j++)
      if (j < nb) v -= B[(long long)j * n + i] * c[j];
    out[i] = v;
    if (z) z[i] = inv_sqrt[i] * v;
  }
}

// y[v] = xp[v] + inv_sqrt[v] * sum_{u in N(v)} z[u]   (z = inv_sqrt * xp);
// 8 lanes per row
__global__ void __launch_bounds__(SP_THREADS)
    spec_spmv(int n, const int* __restrict__ indptr, const int* __restrict__ indices,
              const double* __restrict__ inv_sqrt, const double* __restrict__ xp,
              const double* __restrict__ z, double* __restrict__ y) {
  const int g8 = threadIdx.x & 7;
  const unsigned gmask = 0xffu << (threadIdx.x & 24);
  for (int v = (blockIdx.x * SP_THREADS + threadIdx.x) >> 3; v < n;
       v += (gridDim.x * SP_THREADS) >> 3) {
    const int b = __ldg(indptr + v), e = __ldg(indptr + v + 1);
    double s = 0.0;
    for (int p = b + g8; p < e; p += 8) s += z[__ldg(indices + p)];
    s += __shfl_down_sync(gmask, s, 4, 8);
    s += __shfl_down_sync(gmask, s, 2, 8);
    s += __shfl_down_sync(gmask, s, 1, 8);
    if (g8 == 0) y[v] = xp[v] + inv_sqrt[v] * s;
  }
}

int launch_dots(int n, const double* B, int nb, const double* x, double* partial, double* coef,
                cudaStream_t st) {
  spec_dots_partial<<<SP_DOT_BLOCKS, SP_THREADS, 0, st>>>(n, B, nb, x, partial);
  GU_CHECK_LAUNCH("spec_dots_partial");
  spec_dots_final<<<1, SP_THREADS, 0, st>>>(partial, nb, SP_DOT_BLOCKS, coef);
  GU_CHECK_LAUNCH("spec_dots_final");
  return GU_OK;
}

// ---------------------------------------------------------------- Lanczos
// One thick-restart Lanczos step of layout._top_eigvec on the device, the
// Gram-Schmidt fused into the passes over the basis V (ncv + 1 rows of n):
//   pass 1  y = xp + D^-1/2 A z (the operator's SpMV; xp = P v_j and
//           z = D^-1/2 xp prepared by the previous step) fused with the dots
//           of y against [B; V_0..V_j] (B: the deflated eigenvectors)
//   pass 2  w = y - B c - V h   with c = B^T y and h = V^T y - (V^T B) c,
//           i.e. P y projected against V, fused with the second-pass dots
//           [B; V]^T w (CGS2)
//   pass 3  w -= B c' + V h'   and ||w||^2
//   pass 4  v_{j+1} = w / beta and its dots with B (the row V_{j+1}^T B kept
//           for the next step's h), then xp / z of v_{j+1}
// H[:j+1, j] = h + h', H[j+1, j] = beta are written on the device; every
// reduction is partials per block then one block summing them in a fixed
// order (deterministic).  Replaces four cuBLAS GEMV passes, a norm and a
// scale per step (the torch loop of round 1).
constexpr int LZ_MAX_ROWS = SP_MAX_BASIS + 36;  // B rows + V rows (ncv <= 35)
#ifndef LZ_ACC
#define LZ_ACC 1
#endif
#ifndef LZ_BLOCKS_PER_SM
// lz_rows keeps <= 40 row values per thread (2 CTAs per SM); lz_rows_acc
// also keeps 40 accumulators (1 CTA per SM)
#define LZ_BLOCKS_PER_SM (LZ_ACC ? 1 : 2)
#endif
constexpr int LZ_BLOCKS = 148 * LZ_BLOCKS_PER_SM;  // one wave

struct LzWs {
  double* y;        // n
  double* w;        // n
  double* xp;       // n
  double* z;        // n
  double* partial;  // LZ_MAX_ROWS x LZ_BLOCKS
  double* coef;     // LZ_MAX_ROWS (c | h of the current pass)
  double* hsum;     // LZ_MAX_ROWS (first-pass h kept for H)
  double* beta;     // 1
};

size_t lz_layout(long long n, char* base, LzWs* ws) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = (off + bytes + 255) & ~(size_t)255;
    return o;
  };
  const size_t oy = take(8 * (size_t)n), ow = take(8 * (size_t)n), ox = take(8 * (size_t)n),
               oz = take(8 * (size_t)n), op = take(8 * (size_t)LZ_MAX_ROWS * LZ_BLOCKS),
               oc = take(8 * (size_t)LZ_MAX_ROWS), oh = take(8 * (size_t)LZ_MAX_ROWS),
               ob = take(8);
  if (base && ws) {
    ws->y = (double*)(base + oy);
    ws->w = (double*)(base + ow);
    ws->xp = (double*)(base + ox);
    ws->z = (double*)(base + oz);
    ws->partial = (double*)(base + op);
    ws->coef = (double*)(base + oc);
    ws->hsum = (double*)(base + oh);
    ws->beta = (double*)(base + ob);
  }
  return off;
}

// row r of [B; V]: B_r for r < nb, else V_{r - nb}
__device__ __forceinline__ const double* lz_row(const double* B, int nb, const double* V, long long n,
                                                int r) {
  return r < nb ? B + (long long)r * n : V + (long long)(r - nb) * n;
}

// block-reduce this thread's per-row accumulators acc[q] (row first + q *
// stride; stride 8: the 8-lane groups of a warp hold rows g8, g8 + 8, ...;
// stride 1: every lane holds rows 0, 1, ...) into partial[r][block] for the
// rows r in [r0, r1)
template <int NACC>
__device__ __forceinline__ void lz_block_partials(const double (&acc)[NACC], int first, int stride,
                                                  int r0, int r1, double* partial) {
  __shared__ double sh[LZ_MAX_ROWS][SP_THREADS / 32];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < NACC; q++) {
    double v = acc[q];
    if (stride == 8) {
      v += __shfl_xor_sync(FULL, v, 8);
      v += __shfl_xor_sync(FULL, v, 16);
    } else {
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    }
    const int r = first + q * stride;
    if (r >= r0 && r < r1 && lane < (stride == 8 ? 8 : 1)) sh[r][wid] = v;
  }
  __syncthreads();
  for (int r = r0 + (int)threadIdx.x; r < r1; r += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < SP_THREADS / 32; k++) s += sh[r][k];
    partial[(long long)r * gridDim.x + blockIdx.x] = s;
  }
  __syncthreads();  // sh is reused by the next call
}

// out = x - sum_r row_r * coef_r over the rows of [B; V] (nr of them;
// coef null: out = x), optionally the dots of out with every row (partial
// rows 0..nr-1) and ||out||^2 (partial row nr).  Thread per element: the nr
// row values of element i are loaded coalesced (consecutive threads,
// consecutive i of one row) and kept in registers for the dots, which are
// reduced per warp by butterfly shuffles; lane r & 31 keeps row r's sum.
template <bool DOTS, bool NORM>
__global__ void __launch_bounds__(SP_THREADS, 2)
    lz_rows(int n, const double* __restrict__ B, int nb, const double* __restrict__ V, int nr,
            const double* __restrict__ coef, const double* __restrict__ x,
            double* __restrict__ out, double* __restrict__ partial) {
  __shared__ double c[LZ_MAX_ROWS];
  __shared__ double sh[LZ_MAX_ROWS + 1][SP_THREADS / 32];
  for (int r = threadIdx.x; r < LZ_MAX_ROWS; r += blockDim.x)
    c[r] = (coef && r < nr) ? coef[r] : 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int NA = (LZ_MAX_ROWS + 31) / 32;
  double acc[NA];
#pragma unroll
  for (int q = 0; q < NA; q++) acc[q] = 0.0;
  double nacc = 0.0;
  const int stride = gridDim.x * blockDim.x;
  // block-uniform trip count: every lane reaches the shuffles
  for (int i0 = blockIdx.x * blockDim.x; i0 < n; i0 += stride) {
    const int i = i0 + threadIdx.x;
    const bool ok = i < n;
    double vals[LZ_MAX_ROWS];
#pragma unroll
    for (int r = 0; r < LZ_MAX_ROWS; r++)
      vals[r] = (ok && r < nr) ? __ldg(lz_row(B, nb, V, n, r) + i) : 0.0;
    double o = ok ? x[i] : 0.0;
    if (coef) {
#pragma unroll
      for (int r = 0; r < LZ_MAX_ROWS; r++) o -= vals[r] * c[r];
    }
    if (out && ok) out[i] = o;
    if (DOTS) {
#pragma unroll
      for (int r = 0; r < LZ_MAX_ROWS; r++) {
        if (r < nr) {  // block-uniform
          double s = vals[r] * o;
#pragma unroll
          for (int m = 16; m > 0; m >>= 1) s += __shfl_xor_sync(FULL, s, m);
          if (lane == (r & 31)) acc[r >> 5] += s;
        }
      }
    }
    if (NORM) nacc = fma(o, o, nacc);
  }
  if (DOTS) {
#pragma unroll
    for (int q = 0; q < NA; q++) {
      const int r = q * 32 + lane;
      if (r < nr) sh[r][wid] = acc[q];
    }
  }
  if (NORM) {
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) nacc += __shfl_xor_sync(FULL, nacc, m);
    if (lane == 0) sh[nr][wid] = nacc;
  }
  __syncthreads();
  const int r0 = DOTS ? 0 : nr, r1 = NORM ? nr + 1 : nr;
  for (int r = r0 + (int)threadIdx.x; r < r1; r += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < SP_THREADS / 32; k++) s += sh[r][k];
    partial[(long long)r * gridDim.x + blockIdx.x] = s;
  }
}

// lz_rows with the dots accumulated per thread in registers (one shuffle
// reduction per row at the end instead of per 32 elements): ~2x the
// registers, one CTA per SM, a row pass bound by its loads.  Same
// partial[r][block] contract; the sums' order differs from lz_rows (both
// are fixed, so each is deterministic).
template <bool DOTS, bool NORM, int NRMAX>
__global__ void __launch_bounds__(SP_THREADS, 1)
    lz_rows_acc(int n, const double* __restrict__ B, int nb, const double* __restrict__ V,
                int nr, const double* __restrict__ coef, const double* __restrict__ x,
                double* __restrict__ out, double* __restrict__ partial) {
  __shared__ double c[NRMAX];
  __shared__ double sh[NRMAX + 1][SP_THREADS / 32];
  for (int r = threadIdx.x; r < NRMAX; r += blockDim.x) c[r] = (coef && r < nr) ? coef[r] : 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double acc[NRMAX];
#pragma unroll
  for (int r = 0; r < NRMAX; r++) acc[r] = 0.0;
  double nacc = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double vals[NRMAX];
#pragma unroll
    for (int r = 0; r < NRMAX; r++) vals[r] = r < nr ? __ldg(lz_row(B, nb, V, n, r) + i) : 0.0;
    double o = x[i];
    if (coef) {
#pragma unroll
      for (int r = 0; r < NRMAX; r++) o -= vals[r] * c[r];
    }
    if (out) out[i] = o;
    if (DOTS) {
#pragma unroll
      for (int r = 0; r < NRMAX; r++) acc[r] = fma(vals[r], o, acc[r]);
    }
    if (NORM) nacc = fma(o, o, nacc);
  }
  if (DOTS) {
#pragma unroll
    for (int r = 0; r < NRMAX; r++) {
      double v = acc[r];
      for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(FULL, v, m);
      if (lane == 0 && r < nr) sh[r][wid] = v;
    }
  }
  if (NORM) {
    for (int m = 16; m > 0; m >>= 1) nacc += __shfl_xor_sync(FULL, nacc, m);
    if (lane == 0) sh[nr][wid] = nacc;
  }
  __syncthreads();
  const int r0 = DOTS ? 0 : nr, r1 = NORM ? nr + 1 : nr;
  for (int r = r0 + (int)threadIdx.x; r < r1; r += blockDim.x) {
    double sum = 0.0;
    for (int k = 0; k < SP_THREADS / 32; k++) sum += sh[r][k];
    partial[(long long)r * gridDim.x + blockIdx.x] = sum;
  }
}

// v = w / beta (beta null: v = w, not written); dots of v with B (partials,
// rows 0..nb-1)
__global__ void __launch_bounds__(SP_THREADS)
    lz_scale_dots(int n, const double* __restrict__ w, const double* __restrict__ beta,
                  double* __restrict__ v, const double* __restrict__ B, int nb,
                  double* __restrict__ partial) {
  double acc[SP_MAX_BASIS] = {0.0, 0.0, 0.0, 0.0};
  const double ib = beta ? 1.0 / fmax(*beta, 1e-300) : 1.0;
  for (int i = blockIdx.x * SP_THREADS + threadIdx.x; i < n; i += gridDim.x * SP_THREADS) {
    const double x = w[i] * ib;
    if (v) v[i] = x;
#pragma unroll
    for (int b = 0; b < SP_MAX_BASIS; b++)
      if (b < nb) acc[b] = fma(B[(long long)b * n + i], x, acc[b]);
  }
  lz_block_partials<SP_MAX_BASIS>(acc, 0, 1, 0, nb, partial);
}

// coef[r] = sum_k partial[r][k] in a fixed order, r < nr; mode:
//   0: plain sums into coef (and hsum when save_h)
//   1: first pass: coef = [c | h] with h = V^T y - VB c   (VB: (j+1) x nb)
// One block; rows handled one warp each.
__global__ void lz_final(const double* __restrict__ partial, int nr, int nblocks, int nb,
                         int jrows, const double* __restrict__ VB, int mode,
                         double* __restrict__ coef, double* __restrict__ hsum) {
  __shared__ double s[LZ_MAX_ROWS + 1];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int r = wid; r < nr; r += blockDim.x >> 5) {
    // four independent partial sums per lane (loads in flight together),
    // combined in a fixed order: deterministic
    double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
    const double* pr = partial + (long long)r * nblocks;
    int k = lane;
    for (; k + 96 < nblocks; k += 128) {
      v0 += pr[k];
      v1 += pr[k + 32];
      v2 += pr[k + 64];
      v3 += pr[k + 96];
    }
    for (; k < nblocks; k += 32) v0 += pr[k];
    double v = (v0 + v1) + (v2 + v3);
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(FULL, v, o);
    if (lane == 0) s[r] = v;
  }
  __syncthreads();
  for (int r = threadIdx.x; r < nr; r += blockDim.x) {
    double v = s[r];
    if (mode == 1 && r >= nb) {
      const int i = r - nb;
      for (int b = 0; b < nb; b++) v -= VB[(long long)i * SP_MAX_BASIS + b] * s[b];
    }
    coef[r] = v;
    if (hsum) hsum[r] = v;
  }
}

// H[:j+1, j] = h1 + h2 (rows nb.. of the two coefficient sets), H[j+1, j] =
// beta = sqrt(||w||^2); VB row j+1 = the dots of v_{j+1} with B
__global__ void lz_write_h(const double* __restrict__ hsum, const double* __restrict__ coef2,
                           int nb, int jrows, const double* __restrict__ partial_norm,
                           int nblocks, double* __restrict__ H, int ncv, int j,
                           double* __restrict__ beta) {
  // ||w||^2 from the block partials: strided per-thread sums, then a fixed
  // shuffle / shared tree (deterministic; was one thread's serial loop)
  __shared__ double sw[32];
  double acc = 0.0;
  for (int k = threadIdx.x; k < nblocks; k += blockDim.x) acc += partial_norm[k];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(FULL, acc, o);
  if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) s += sw[w];
    const double bt = sqrt(s);
    *beta = bt;
    H[(long long)(j + 1) * ncv + j] = bt;
  }
  for (int i = threadIdx.x; i < jrows; i += blockDim.x)
    H[(long long)i * ncv + j] = hsum[nb + i] + coef2[nb + i];
}

// xp = v - B vb, z = inv_sqrt * xp (the next operator input)
__global__ void lz_prepare(int n, const double* __restrict__ v, const double* __restrict__ B,
                           int nb, const double* __restrict__ vb,
                           const double* __restrict__ inv_sqrt, double* __restrict__ xp,
                           double* __restrict__ z) {
  double c[SP_MAX_BASIS];
#pragma unroll
  for (int b = 0; b < SP_MAX_BASIS; b++) c[b] = b < nb ? vb[b] : 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double x = v[i];
#pragma unroll
    for (int b = 0; b < SP_MAX_BASIS; b++)
      if (b < nb) x -= B[(long long)b * n + i] * c[b];
    xp[i] = x;
    z[i] = inv_sqrt[i] * x;
  }
}

}  // namespace
}  // namespace gu

using namespace gu;

extern "C" int gu_spectral_degree(int64_t n, const int32_t* indptr, double* inv_sqrt,
                                  double* sqrt_deg, void* stream) {
  if (n < 1 || n >= INT_MAX) {
    set_error("gu_spectral_degree: n=%lld", (long long)n);
    return GU_ERR_ARG;
  }
  spec_degree<<<148 * 4, SP_THREADS, 0, (cudaStream_t)stream>>>((int)n, indptr, inv_sqrt, sqrt_deg);
  GU_CHECK_LAUNCH("spec_degree");
  return GU_OK;
}

extern "C" size_t gu_spectral_op_workspace_size(int64_t n) {
  return sizeof(double) * (2 * (size_t)n + (size_t)SP_MAX_BASIS * SP_DOT_BLOCKS + 2 * SP_MAX_BASIS);
}

// y = P (x' + D^-1/2 A D^-1/2 x'), x' = P x, P = I - B B^T; basis: nb <= 4
// orthonormal float64 columns, column j at basis + j*n.  x and y may not alias.
extern "C" int gu_spectral_op(int64_t n, const int32_t* indptr, const int32_t* indices,
                              const double* inv_sqrt, const double* basis, int32_t nb,
                              const double* x, double* y, void* workspace, size_t ws_bytes,
                              void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 1 || n >= INT_MAX || nb < 0 || nb > SP_MAX_BASIS || x == y) {
    set_error("gu_spectral_op: bad arguments (n=%lld nb=%d)", (long long)n, nb);
    return GU_ERR_ARG;
  }
  if (!workspace || ws_bytes < gu_spectral_op_workspace_size(n)) {
    set_error("gu_spectral_op: workspace too small");
    return GU_ERR_WORKSPACE;
  }
  double* xp = (double*)workspace;
  double* z = xp + n;
  double* partial = z + n;
  double* c1 = partial + SP_MAX_BASIS * SP_DOT_BLOCKS;
  double* c2 = c1 + SP_MAX_BASIS;
  const int N = (int)n;
  if (nb > 0) {
    int rc = launch_dots(N, basis, nb, x, partial, c1, st);
    if (rc != GU_OK) return rc;
  }
  spec_project<<<148 * 4, SP_THREADS, 0, st>>>(N, basis, nb, c1, x, xp, inv_sqrt, z);
  GU_CHECK_LAUNCH("spec_project");
  const long long rows_per_block = SP_THREADS / 8;
  long long blocks = (n + rows_per_block - 1) / rows_per_block;
  if (blocks > 148 * 16) blocks = 148 * 16;
  spec_spmv<<<(unsigned)blocks, SP_THREADS, 0, st>>>(N, indptr, indices, inv_sqrt, xp, z, y);
  GU_CHECK_LAUNCH("spec_spmv");
  if (nb > 0) {
    int rc = launch_dots(N, basis, nb, y, partial, c2, st);
    if (rc != GU_OK) return rc;
    spec_project<<<148 * 4, SP_THREADS, 0, st>>>(N, basis, nb, c2, y, y, inv_sqrt, nullptr);
    GU_CHECK_LAUNCH("spec_project");
  }
  return GU_OK;
}

extern "C" size_t gu_lanczos_workspace_size(int64_t n) { return lz_layout(n, nullptr, nullptr); }

// vb (device, nb doubles) = B^T v, and the operator input (xp, z) of v kept
// in the workspace for the next gu_lanczos_step.
extern "C" int gu_lanczos_prepare(int64_t n, const double* inv_sqrt, const double* basis,
                                  int32_t nb, const double* v, double* vb, void* workspace,
                                  size_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 1 || n >= INT_MAX || nb < 0 || nb > SP_MAX_BASIS) {
    set_error("gu_lanczos_prepare: bad arguments");
    return GU_ERR_ARG;
  }
  LzWs ws;
  if (!workspace || ws_bytes < lz_layout(n, (char*)workspace, &ws)) {
    set_error("gu_lanczos_prepare: workspace too small");
    return GU_ERR_WORKSPACE;
  }
  const int N = (int)n;
  if (nb > 0) {  // vb = B^T v
    lz_scale_dots<<<LZ_BLOCKS, SP_THREADS, 0, st>>>(N, v, nullptr, nullptr, basis, nb,
                                                    ws.partial);
    GU_CHECK_LAUNCH("lz_scale_dots");
    lz_final<<<1, SP_THREADS, 0, st>>>(ws.partial, nb, LZ_BLOCKS, nb, 0, nullptr, 0, vb, nullptr);
    GU_CHECK_LAUNCH("lz_final");
  }
  lz_prepare<<<LZ_BLOCKS, SP_THREADS, 0, st>>>(N, v, basis, nb, vb, inv_sqrt, ws.xp, ws.z);
  GU_CHECK_LAUNCH("lz_prepare");
  return GU_OK;
}

// One Lanczos step j (see the kernels above).  V: (ncv + 1) x n row-major,
// rows 0..j filled, row j's operator input prepared (gu_lanczos_prepare or
// the previous step); VB: (ncv + 1) x 4 row-major, rows 0..j = V_i^T B;
// H: (ncv + 1) x ncv row-major.  Writes V row j + 1, VB row j + 1, H[:j+2, j]
// and prepares row j + 1's operator input.  No host synchronisation.
extern "C" int gu_lanczos_step(int64_t n, const int32_t* indptr, const int32_t* indices,
                               const double* inv_sqrt, const double* basis, int32_t nb,
                               double* V, double* VB, double* H, int32_t ncv, int32_t j,
                               void* workspace, size_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 1 || n >= INT_MAX || nb < 0 || nb > SP_MAX_BASIS || ncv < 1 ||
      ncv + 1 + SP_MAX_BASIS > LZ_MAX_ROWS || j < 0 || j >= ncv) {
    set_error("gu_lanczos_step: bad arguments (n=%lld nb=%d ncv=%d j=%d)", (long long)n, nb,
              ncv, j);
    return GU_ERR_ARG;
  }
  LzWs ws;
  if (!workspace || ws_bytes < lz_layout(n, (char*)workspace, &ws)) {
    set_error("gu_lanczos_step: workspace too small");
    return GU_ERR_WORKSPACE;
  }
  const int N = (int)n;
  const int jrows = j + 1, nr = nb + jrows;
  const long long rows_per_block = SP_THREADS / 8;
  long long sblocks = (n + rows_per_block - 1) / rows_per_block;
  if (sblocks > 148 * 16) sblocks = 148 * 16;
  // pass 1: y = operator(v_j), then the dots [B; V]^T y
  spec_spmv<<<(unsigned)sblocks, SP_THREADS, 0, st>>>(N, indptr, indices, inv_sqrt, ws.xp, ws.z,
                                                      ws.y);
  GU_CHECK_LAUNCH("spec_spmv");
  const bool acc_mode = LZ_ACC;
  if (acc_mode)
    lz_rows_acc<true, false, LZ_MAX_ROWS><<<LZ_BLOCKS, SP_THREADS, 0, st>>>(
        N, basis, nb, V, nr, nullptr, ws.y, nullptr, ws.partial);
  else
    lz_rows<true, false><<<LZ_BLOCKS, SP_THREADS, 0, st>>>(N, basis, nb, V, nr, nullptr, ws.y,
                                                           nullptr, ws.partial);
  GU_CHECK_LAUNCH("lz_rows");
  lz_final<<<1, SP_THREADS, 0, st>>>(ws.partial, nr, LZ_BLOCKS, nb, jrows, VB, 1, ws.coef,
                                     ws.hsum);
  GU_CHECK_LAUNCH("lz_final");
  // pass 2: w = y - B c - V h, dots [B; V]^T w
  if (acc_mode)
    lz_rows_acc<true, false, LZ_MAX_ROWS><<<LZ_BLOCKS, SP_THREADS, 0, st>>>(
        N, basis, nb, V, nr, ws.coef, ws.y, ws.w, ws.partial);
  else
  lz_rows<true, false><<<LZ_BLOCKS, SP_THREADS, 0, st>>>(N, basis, nb, V, nr, ws.coef, ws.y,
                                                         ws.w, ws.partial);
  GU_CHECK_LAUNCH("lz_rows");
  lz_final<<<1, SP_THREADS, 0, st>>>(ws.partial, nr, LZ_BLOCKS, nb, jrows, nullptr, 0, ws.coef,
                                     nullptr);
  GU_CHECK_LAUNCH("lz_final");
  // pass 3: w -= B c' + V h', ||w||^2 (partial row nr)
  if (acc_mode)
    lz_rows_acc<false, true, LZ_MAX_ROWS><<<LZ_BLOCKS, SP_THREADS, 0, st>>>(
        N, basis, nb, V, nr, ws.coef, ws.w, ws.w, ws.partial);
  else
  lz_rows<false, true><<<LZ_BLOCKS, SP_THREADS, 0, st>>>(N, basis, nb, V, nr, ws.coef, ws.w,
                                                         ws.w, ws.partial);
  GU_CHECK_LAUNCH("lz_rows");
  lz_write_h<<<1, SP_THREADS, 0, st>>>(ws.hsum, ws.coef, nb, jrows,
                                       ws.partial + (long long)nr * LZ_BLOCKS, LZ_BLOCKS, H, ncv,
                                       j, ws.beta);
  GU_CHECK_LAUNCH("lz_write_h");
  // pass 4: v_{j+1} = w / beta, its dots with B, then its operator input
  double* vnext = V + (long long)(j + 1) * n;
  double* vbnext = VB + (long long)(j + 1) * SP_MAX_BASIS;
  lz_scale_dots<<<LZ_BLOCKS, SP_THREADS, 0, st>>>(N, ws.w, ws.beta, vnext, basis, nb, ws.partial);
  GU_CHECK_LAUNCH("lz_scale_dots");
  if (nb > 0) {
    lz_final<<<1, SP_THREADS, 0, st>>>(ws.partial, nb, LZ_BLOCKS, nb, 0, nullptr, 0, vbnext,
                                       nullptr);
    GU_CHECK_LAUNCH("lz_final");
  }
  lz_prepare<<<LZ_BLOCKS, SP_THREADS, 0, st>>>(N, vnext, basis, nb, vbnext, inv_sqrt, ws.xp, ws.z);
  GU_CHECK_LAUNCH("lz_prepare");
  return GU_OK;
}
