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
