// capi.cu -- library-level C ABI: errors, version, sync, record packing.
#include <cstdarg>
#include <cstdio>

#include "common.cuh"
#include "gumap.h"

namespace gu {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char* what) {
  set_error("%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
  return GU_ERR_CUDA;
}

namespace {

constexpr int SCAN_THREADS = 1024;
constexpr int SCAN_ITEMS = 4;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

__device__ __forceinline__ long long block_excl_scan(long long v, long long* sh, long long* total) {
  // sh: 32 slots
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long inc = warp_incl_scan(v);
  if (lane == 31) sh[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    long long x = (lane < (int)(blockDim.x >> 5)) ? sh[lane] : 0;
    long long xi = warp_incl_scan(x);
    sh[lane] = xi - x;
    if (lane == 31) sh[32] = xi;
  }
  __syncthreads();
  long long r = sh[warp] + inc - v;
  *total = sh[32];
  __syncthreads();
  return r;
}

__global__ void scan_tile_sums(const int* __restrict__ cnt, long long nrows, long long* partial) {
  __shared__ long long sh[33];
  long long base = (long long)blockIdx.x * SCAN_TILE;
  long long s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) {
    long long r = base + (long long)threadIdx.x * SCAN_ITEMS + i;
    if (r < nrows) s += cnt[r];
  }
  long long total;
  block_excl_scan(s, sh, &total);
  if (threadIdx.x == 0) partial[blockIdx.x] = total;
}

__global__ void scan_partials(long long* partial, long long nparts) {
  __shared__ long long sh[33];
  long long carry = 0;
  for (long long b = 0; b < nparts; b += SCAN_THREADS) {
    long long i = b + threadIdx.x;
    long long v = i < nparts ? partial[i] : 0;
    long long total;
    long long ex = block_excl_scan(v, sh, &total);
    if (i < nparts) partial[i] = carry + ex;
    carry += total;
  }
  if (threadIdx.x == 0) partial[nparts] = carry;
}

__global__ void scan_tiles_write(const int* __restrict__ cnt, long long nrows,
                                 const long long* __restrict__ partial, long long* indptr) {
  __shared__ long long sh[33];
  long long base = (long long)blockIdx.x * SCAN_TILE;
  long long v[SCAN_ITEMS];
  long long s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) {
    long long r = base + (long long)threadIdx.x * SCAN_ITEMS + i;
    v[i] = r < nrows ? cnt[r] : 0;
    s += v[i];
  }
  long long total;
  long long ex = block_excl_scan(s, sh, &total) + partial[blockIdx.x];
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) {
    long long r = base + (long long)threadIdx.x * SCAN_ITEMS + i;
    if (r < nrows) indptr[r] = ex;
    ex += v[i];
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
    indptr[nrows] = partial[gridDim.x];
  }
}

__global__ void pack_rows(long long nrows, int k, const int* __restrict__ rn,
                          const int* __restrict__ rd, const int* __restrict__ rc,
                          const long long* __restrict__ indptr, int* __restrict__ od,
                          int* __restrict__ odist) {
  long long total = nrows * (long long)k;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    long long r = i / k;
    int j = (int)(i - r * k);
    if (j < rc[r]) {
      long long o = indptr[r] + j;
      od[o] = rn[i];
      odist[o] = rd[i];
    }
  }
}

}  // namespace

// exclusive scan of int32 counts -> int64 indptr[nrows+1] (used by several ops)
int scan_counts(const int* cnt, long long nrows, long long* indptr, long long* partial,
                cudaStream_t st) {
  if (nrows == 0) {
    GU_CHECK(cudaMemsetAsync(indptr, 0, sizeof(long long), st));
    return GU_OK;
  }
  long long tiles = (nrows + SCAN_TILE - 1) / SCAN_TILE;
  scan_tile_sums<<<(unsigned)tiles, SCAN_THREADS, 0, st>>>(cnt, nrows, partial);
  GU_CHECK_LAUNCH("scan_tile_sums");
  scan_partials<<<1, SCAN_THREADS, 0, st>>>(partial, tiles);
  GU_CHECK_LAUNCH("scan_partials");
  scan_tiles_write<<<(unsigned)tiles, SCAN_THREADS, 0, st>>>(cnt, nrows, partial, indptr);
  GU_CHECK_LAUNCH("scan_tiles_write");
  return GU_OK;
}

size_t scan_workspace(long long nrows) {
  return sizeof(long long) * (size_t)((nrows + SCAN_TILE - 1) / SCAN_TILE + 1);
}

}  // namespace gu

using namespace gu;

namespace gu {
namespace {
// numpy Generator(PCG64(SeedSequence(seed))).uniform(low, high, count):
// element f = low + (high - low) * ((next_uint64 >> 11) * 2^-53) of the f-th
// draw (numpy distributions.c random_uniform / next_double; no FMA).  Each
// thread jumps its generator to its first element (pcg64_advance) and walks
// a run of consecutive elements.
constexpr int RU_RUN = 64;
__global__ void random_uniform_kernel(long long count, unsigned long long seed, double low,
                                      double range, double* __restrict__ out) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long f0 = t * RU_RUN;
  if (f0 >= count) return;
  Pcg64 r;
  pcg64_from_seedseq(r, seed, 0, false);
  pcg64_advance(r, (unsigned long long)f0);
  const long long f1 = f0 + RU_RUN < count ? f0 + RU_RUN : count;
  for (long long f = f0; f < f1; f++) {
    const double d = (double)(r.next64() >> 11) * (1.0 / 9007199254740992.0);
    out[f] = __dadd_rn(low, __dmul_rn(range, d));
  }
}
}  // namespace
}  // namespace gu

extern "C" int gu_random_uniform(int64_t count, uint64_t seed, double low, double high,
                                 double* out, void* stream) {
  if (count < 0) {
    gu::set_error("gu_random_uniform: negative count");
    return GU_ERR_ARG;
  }
  if (count == 0) return GU_OK;
  const long long threads = (count + gu::RU_RUN - 1) / gu::RU_RUN;
  gu::random_uniform_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      count, seed, low, high - low, out);
  GU_CHECK_LAUNCH("random_uniform_kernel");
  return GU_OK;
}

extern "C" int gu_version(void) { return 1; }
extern "C" const char* gu_last_error(void) { return g_err; }

extern "C" int gu_device_sync(void* stream) {
  GU_CHECK(cudaStreamSynchronize((cudaStream_t)stream));
  GU_CHECK(cudaGetLastError());
  return GU_OK;
}

extern "C" int gu_host_is_pinned(const void* ptr) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();  // unregistered pageable memory on old drivers: clear it
    return 0;
  }
  return a.type == cudaMemoryTypeHost ? 1 : 0;
}

extern "C" size_t gu_pack_records_workspace_size(int64_t nrows) { return scan_workspace(nrows); }

extern "C" int gu_pack_records(int64_t nrows, int32_t k, const int32_t* rec_nbr,
                               const int32_t* rec_dist, const int32_t* rec_count,
                               int64_t* out_indptr, int32_t* out_dst, int32_t* out_dist,
                               void* workspace, size_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (nrows < 0 || k < 0) {
    set_error("gu_pack_records: bad arguments");
    return GU_ERR_ARG;
  }
  if (ws_bytes < scan_workspace(nrows)) {
    set_error("gu_pack_records: workspace too small");
    return GU_ERR_WORKSPACE;
  }
  int r = scan_counts(rec_count, nrows, (long long*)out_indptr, (long long*)workspace, st);
  if (r) return r;
  if (nrows == 0 || k == 0) return GU_OK;
  long long total = nrows * (long long)k;
  unsigned blocks = (unsigned)((total + 255) / 256 < 148LL * 64 ? (total + 255) / 256 : 148LL * 64);
  pack_rows<<<blocks, 256, 0, st>>>(nrows, k, rec_nbr, rec_dist, rec_count,
                                    (const long long*)out_indptr, out_dst, out_dist);
  GU_CHECK_LAUNCH("pack_rows");
  return GU_OK;
}
