// ingest.cu -- graph construction and LCC extraction on the GPU (SURVEY 8(f)
// row 4; /root/reference/pkg/src/graph_umap/graph.py:114-232).
//
//   build_graph                 graph.py:132-186  dense relabel by sorted id,
//       drop self loops, dedupe, canonical u < v edges in (u, v) order, CSR of
//       both orientations with sorted adjacency (_from_canonical, 114-129)
//   largest_connected_component graph.py:201-232  largest component (ties:
//       the one holding the smallest vertex), dense relabel in id order
// All sorts are CUB radix sorts of 64-bit keys; compaction preserves order.
#include <climits>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include "common.cuh"
#include "gumap.h"

namespace gu {
namespace {

constexpr int IG_THREADS = 256;
constexpr int IG_BLOCKS = 148 * 8;

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

struct Carve {
  char* base;
  size_t off = 0;
  template <class T>
  T* take(size_t count) {
    T* p = base ? (T*)(base + off) : nullptr;
    off = align256(off + sizeof(T) * (count ? count : 1));
    return p;
  }
};

// dense id of each endpoint (binary search in the sorted unique ids), then
// the canonical key (min << 32 | max); self loops get the sentinel ~0
__global__ void ig_relabel(long long np2, const long long* __restrict__ raw,
                           const long long* __restrict__ ids, int n,
                           unsigned long long* __restrict__ key, int* __restrict__ loops) {
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < np2 / 2;
       p += (long long)gridDim.x * blockDim.x) {
    int d[2];
#pragma unroll
    for (int s = 0; s < 2; s++) {
      const long long x = raw[2 * p + s];
      int lo = 0, hi = n - 1;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (ids[mid] < x) lo = mid + 1;
        else hi = mid;
      }
      d[s] = lo;
    }
    if (d[0] == d[1]) {
      key[p] = ~0ull;
      atomicAdd(loops, 1);
    } else {
      const unsigned a = (unsigned)min(d[0], d[1]), b = (unsigned)max(d[0], d[1]);
      key[p] = ((unsigned long long)a << 32) | b;
    }
  }
}

// both orientations of each canonical edge key, and the degree counts
__global__ void ig_both(long long m, const unsigned long long* __restrict__ key,
                        unsigned long long* __restrict__ both, long long* __restrict__ deg) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += (long long)gridDim.x * blockDim.x) {
    const unsigned long long k = key[e];
    const unsigned a = (unsigned)(k >> 32), b = (unsigned)k;
    both[2 * e] = k;
    both[2 * e + 1] = ((unsigned long long)b << 32) | a;
    atomicAdd((unsigned long long*)(deg + a), 1ull);
    atomicAdd((unsigned long long*)(deg + b), 1ull);
  }
}

__global__ void ig_unpack(long long m, const unsigned long long* __restrict__ key,
                          long long* __restrict__ edges, const unsigned long long* __restrict__ both,
                          int* __restrict__ indices) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < 2 * m;
       e += (long long)gridDim.x * blockDim.x) {
    if (e < m) {
      edges[2 * e] = (long long)(key[e] >> 32);
      edges[2 * e + 1] = (long long)(unsigned)key[e];
    }
    indices[e] = (int)(unsigned)both[e];
  }
}

// ---- LCC
__global__ void ig_sizes(int n, const int* __restrict__ label, int* __restrict__ size) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    atomicAdd(size + label[v], 1);
}

// champion = max size, ties to the smallest label (= smallest vertex id)
__global__ void ig_champion(int n, const int* __restrict__ size, unsigned long long* best) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const int s = size[v];
    if (s > 0)
      atomicMax(best, ((unsigned long long)(unsigned)s << 32) | (unsigned)(INT_MAX - v));
  }
}

__global__ void ig_keep_flags(int n, const int* __restrict__ label,
                              const unsigned long long* __restrict__ best, int* __restrict__ keep) {
  const int champ = INT_MAX - (int)(unsigned)(*best);
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    keep[v] = label[v] == champ ? 1 : 0;
}

// edges of the champion, remapped (order kept: the remap is monotone)
__global__ void ig_lcc_keys(long long m, const long long* __restrict__ edges,
                            const int* __restrict__ keep, const int* __restrict__ remap,
                            unsigned long long* __restrict__ key, unsigned char* __restrict__ flag) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += (long long)gridDim.x * blockDim.x) {
    const int u = (int)edges[2 * e], v = (int)edges[2 * e + 1];
    const bool k = keep[u] != 0;
    flag[e] = k ? 1 : 0;
    key[e] = k ? (((unsigned long long)(unsigned)remap[u] << 32) | (unsigned)remap[v]) : 0ull;
  }
}

__global__ void ig_kept_ids(int n, const int* __restrict__ keep, const int* __restrict__ remap,
                            int* __restrict__ old_of_new) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    if (keep[v]) old_of_new[remap[v]] = v;
}

int bits_for(long long n) {
  int b = 1;
  while (b < 32 && (1ll << b) < n) b++;
  return b;
}

// canonical sorted keys (m_c of them, unique) -> edges, CSR.  deg: n+1
// int64 zeroed; both: 2 m_c keys (scratch); indptr n+1; indices 2 m_c.
int keys_to_graph(long long n, long long mc, const unsigned long long* keys, unsigned long long* both,
                  unsigned long long* both_sorted, long long* deg, long long* edges,
                  long long* indptr, int* indices, void* tmp, size_t tmp_bytes, cudaStream_t st) {
  GU_CHECK(cudaMemsetAsync(deg, 0, sizeof(long long) * (size_t)(n + 1), st));
  if (mc > 0) {
    ig_both<<<IG_BLOCKS, IG_THREADS, 0, st>>>(mc, keys, both, deg);
    GU_CHECK_LAUNCH("ig_both");
    const int vb = bits_for(n);
    size_t tb = tmp_bytes;
    GU_CHECK(cub::DeviceRadixSort::SortKeys(tmp, tb, both, both_sorted, (int)(2 * mc), 0, 32 + vb, st));
    ig_unpack<<<IG_BLOCKS, IG_THREADS, 0, st>>>(mc, keys, edges, both_sorted, indices);
    GU_CHECK_LAUNCH("ig_unpack");
  }
  size_t tb = tmp_bytes;
  GU_CHECK(cub::DeviceScan::ExclusiveSum(tmp, tb, deg, indptr, (int)(n + 1), st));
  return GU_OK;
}

size_t sort_tmp_bytes(long long count) {
  size_t a = 0, b = 0, c = 0, d = 0;
  const int cnt = (int)(count > 0 ? count : 1);
  cub::DeviceRadixSort::SortKeys(nullptr, a, (const unsigned long long*)nullptr,
                                 (unsigned long long*)nullptr, cnt);
  cub::DeviceSelect::Unique(nullptr, b, (const unsigned long long*)nullptr,
                            (unsigned long long*)nullptr, (int*)nullptr, cnt);
  cub::DeviceScan::ExclusiveSum(nullptr, c, (const long long*)nullptr, (long long*)nullptr, cnt);
  cub::DeviceSelect::Flagged(nullptr, d, (const unsigned long long*)nullptr,
                             (const unsigned char*)nullptr, (unsigned long long*)nullptr,
                             (int*)nullptr, cnt);
  size_t x = a > b ? a : b;
  x = x > c ? x : c;
  return x > d ? x : d;
}

}  // namespace
}  // namespace gu

using namespace gu;

// ---------------------------------------------------------- build_graph
// Phase 1 (gu_build_graph_ids): sorted unique ids of the raw pairs -> n.
// Phase 2 (gu_build_graph_csr): canonical edges + CSR into caller buffers
// sized from n and the returned edge count.
extern "C" size_t gu_build_graph_workspace_size(int64_t npairs) {
  Carve c{nullptr};
  c.take<long long>((size_t)(2 * npairs));           // sorted raw ids
  c.take<long long>((size_t)(2 * npairs));           // unique ids
  c.take<int>(2);                                    // counts
  c.take<unsigned long long>((size_t)npairs);        // keys
  c.take<unsigned long long>((size_t)npairs);        // sorted keys
  c.take<unsigned long long>((size_t)npairs);        // unique keys
  c.take<unsigned long long>((size_t)(2 * npairs));  // both
  c.take<unsigned long long>((size_t)(2 * npairs));  // both sorted
  c.take<long long>((size_t)(2 * npairs) + 1);       // degrees (n <= 2 npairs)
  c.take<char>(sort_tmp_bytes(2 * npairs));
  return c.off;
}

struct BuildWs {
  long long *raw_sorted, *ids;
  int* counts;
  unsigned long long *keys, *keys_sorted, *keys_unique, *both, *both_sorted;
  long long* deg;
  void* tmp;
  size_t tmp_bytes;
};

static BuildWs build_ws(int64_t npairs, char* base) {
  Carve c{base};
  BuildWs w;
  w.raw_sorted = c.take<long long>((size_t)(2 * npairs));
  w.ids = c.take<long long>((size_t)(2 * npairs));
  w.counts = c.take<int>(2);
  w.keys = c.take<unsigned long long>((size_t)npairs);
  w.keys_sorted = c.take<unsigned long long>((size_t)npairs);
  w.keys_unique = c.take<unsigned long long>((size_t)npairs);
  w.both = c.take<unsigned long long>((size_t)(2 * npairs));
  w.both_sorted = c.take<unsigned long long>((size_t)(2 * npairs));
  w.deg = c.take<long long>((size_t)(2 * npairs) + 1);
  w.tmp_bytes = sort_tmp_bytes(2 * npairs);
  w.tmp = c.take<char>(w.tmp_bytes);
  return w;
}

// raw: int64 (npairs, 2) non-negative ids on the device.  host_out[0] = n,
// host_out[1] = canonical edge count m, host_out[2] = self loops dropped.
extern "C" int gu_build_graph_ids(int64_t npairs, const int64_t* raw, int64_t* host_out,
                                  void* workspace, size_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (npairs < 1 || 2 * npairs >= INT_MAX) {
    set_error("gu_build_graph: %lld pairs out of range", (long long)npairs);
    return GU_ERR_ARG;
  }
  if (!workspace || ws_bytes < gu_build_graph_workspace_size(npairs)) {
    set_error("gu_build_graph: workspace too small");
    return GU_ERR_WORKSPACE;
  }
  BuildWs w = build_ws(npairs, (char*)workspace);
  const int cnt2 = (int)(2 * npairs);
  size_t tb = w.tmp_bytes;
  GU_CHECK(cub::DeviceRadixSort::SortKeys(w.tmp, tb, (const unsigned long long*)raw,
                                          (unsigned long long*)w.raw_sorted, cnt2, 0, 64, st));
  tb = w.tmp_bytes;
  GU_CHECK(cub::DeviceSelect::Unique(w.tmp, tb, (const unsigned long long*)w.raw_sorted,
                                     (unsigned long long*)w.ids, w.counts, cnt2, st));
  int n = 0;
  GU_CHECK(cudaMemcpyAsync(&n, w.counts, sizeof(int), cudaMemcpyDeviceToHost, st));
  GU_CHECK(cudaMemsetAsync(w.counts + 1, 0, sizeof(int), st));
  GU_CHECK(cudaStreamSynchronize(st));
  ig_relabel<<<IG_BLOCKS, IG_THREADS, 0, st>>>(2 * npairs, (const long long*)raw, w.ids, n, w.keys, w.counts + 1);
  GU_CHECK_LAUNCH("ig_relabel");
  const int vb = bits_for(n);
  tb = w.tmp_bytes;
  GU_CHECK(cub::DeviceRadixSort::SortKeys(w.tmp, tb, w.keys, w.keys_sorted, (int)npairs, 0, 64, st));
  tb = w.tmp_bytes;
  GU_CHECK(cub::DeviceSelect::Unique(w.tmp, tb, w.keys_sorted, w.keys_unique, w.counts, (int)npairs, st));
  int uniq = 0, loops = 0;
  GU_CHECK(cudaMemcpyAsync(&uniq, w.counts, sizeof(int), cudaMemcpyDeviceToHost, st));
  GU_CHECK(cudaMemcpyAsync(&loops, w.counts + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  GU_CHECK(cudaStreamSynchronize(st));
  (void)vb;
  // the loop sentinel ~0 sorts last and is unique: drop it
  host_out[0] = n;
  host_out[1] = uniq - (loops > 0 ? 1 : 0);
  host_out[2] = loops;
  return GU_OK;
}

// after gu_build_graph_ids on the same workspace: ids (int64 n), edges (int64
// (m, 2)), indptr (int64 n+1), indices (int32 2m) into caller buffers
extern "C" int gu_build_graph_csr(int64_t npairs, int64_t n, int64_t m, int64_t* out_ids,
                                  int64_t* out_edges, int64_t* out_indptr, int32_t* out_indices,
                                  void* workspace, size_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!workspace || ws_bytes < gu_build_graph_workspace_size(npairs) || m < 0 || n < 1) {
    set_error("gu_build_graph_csr: bad arguments");
    return GU_ERR_ARG;
  }
  BuildWs w = build_ws(npairs, (char*)workspace);
  GU_CHECK(cudaMemcpyAsync(out_ids, w.ids, sizeof(long long) * (size_t)n, cudaMemcpyDeviceToDevice, st));
  return keys_to_graph(n, m, w.keys_unique, w.both, w.both_sorted, w.deg, (long long*)out_edges,
                       (long long*)out_indptr,
                       out_indices, w.tmp, w.tmp_bytes, st);
}

// ------------------------------------------------------------------ LCC
extern "C" size_t gu_lcc_workspace_size(int64_t n, int64_t m) {
  Carve c{nullptr};
  c.take<int>((size_t)n);                      // labels
  c.take<int>((size_t)n);                      // uf scratch
  c.take<int>((size_t)n);                      // sizes
  c.take<unsigned long long>(1);               // champion
  c.take<int>((size_t)n);                      // keep
  c.take<int>((size_t)n + 1);                  // remap
  c.take<int>(2);                              // counts
  c.take<unsigned long long>((size_t)m);       // keys
  c.take<unsigned char>((size_t)m);            // flags
  c.take<unsigned long long>((size_t)m);       // kept keys
  c.take<unsigned long long>((size_t)(2 * m)); // both
  c.take<unsigned long long>((size_t)(2 * m)); // both sorted
  c.take<long long>((size_t)n + 1);            // degrees
  size_t t = sort_tmp_bytes(2 * m > n + 1 ? 2 * m : n + 1);
  c.take<char>(t);
  return c.off;
}

struct LccWs {
  int *labels, *uf, *sizes;
  unsigned long long* best;
  int *keep, *remap, *counts;
  unsigned long long* keys;
  unsigned char* flags;
  unsigned long long *kept, *both, *both_sorted;
  long long* deg;
  void* tmp;
  size_t tmp_bytes;
};

static LccWs lcc_ws(int64_t n, int64_t m, char* base) {
  Carve c{base};
  LccWs w;
  w.labels = c.take<int>((size_t)n);
  w.uf = c.take<int>((size_t)n);
  w.sizes = c.take<int>((size_t)n);
  w.best = c.take<unsigned long long>(1);
  w.keep = c.take<int>((size_t)n);
  w.remap = c.take<int>((size_t)n + 1);
  w.counts = c.take<int>(2);
  w.keys = c.take<unsigned long long>((size_t)m);
  w.flags = c.take<unsigned char>((size_t)m);
  w.kept = c.take<unsigned long long>((size_t)m);
  w.both = c.take<unsigned long long>((size_t)(2 * m));
  w.both_sorted = c.take<unsigned long long>((size_t)(2 * m));
  w.deg = c.take<long long>((size_t)n + 1);
  w.tmp_bytes = sort_tmp_bytes(2 * m > n + 1 ? 2 * m : n + 1);
  w.tmp = c.take<char>(w.tmp_bytes);
  return w;
}

// phase 1: components; host_out[0] = components, [1] = champion size n2,
// [2] = champion edges m2
extern "C" int gu_lcc_plan(int64_t n, int64_t m, const int32_t* indptr, const int32_t* indices,
                           const int64_t* edges, int64_t* host_out, void* workspace,
                           size_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 1 || n >= INT_MAX || m < 0 || 2 * m >= INT_MAX) {
    set_error("gu_lcc_plan: bad arguments");
    return GU_ERR_ARG;
  }
  if (!workspace || ws_bytes < gu_lcc_workspace_size(n, m)) {
    set_error("gu_lcc_plan: workspace too small");
    return GU_ERR_WORKSPACE;
  }
  LccWs w = lcc_ws(n, m, (char*)workspace);
  int rc = gu_connected_components(n, indptr, indices, w.labels, w.counts, w.uf,
                                   sizeof(int) * (size_t)n, stream);
  if (rc != GU_OK) return rc;
  int ncomp = 0;
  GU_CHECK(cudaMemcpyAsync(&ncomp, w.counts, sizeof(int), cudaMemcpyDeviceToHost, st));
  GU_CHECK(cudaMemsetAsync(w.sizes, 0, sizeof(int) * (size_t)n, st));
  GU_CHECK(cudaMemsetAsync(w.best, 0, sizeof(unsigned long long), st));
  ig_sizes<<<IG_BLOCKS, IG_THREADS, 0, st>>>((int)n, w.labels, w.sizes);
  GU_CHECK_LAUNCH("ig_sizes");
  ig_champion<<<IG_BLOCKS, IG_THREADS, 0, st>>>((int)n, w.sizes, w.best);
  GU_CHECK_LAUNCH("ig_champion");
  ig_keep_flags<<<IG_BLOCKS, IG_THREADS, 0, st>>>((int)n, w.labels, w.best, w.keep);
  GU_CHECK_LAUNCH("ig_keep_flags");
  size_t tb = w.tmp_bytes;
  GU_CHECK(cub::DeviceScan::ExclusiveSum(w.tmp, tb, w.keep, w.remap, (int)n, st));
  if (m > 0) {
    ig_lcc_keys<<<IG_BLOCKS, IG_THREADS, 0, st>>>(m, (const long long*)edges, w.keep, w.remap,
                                                  w.keys, w.flags);
    GU_CHECK_LAUNCH("ig_lcc_keys");
    tb = w.tmp_bytes;
    GU_CHECK(cub::DeviceSelect::Flagged(w.tmp, tb, w.keys, w.flags, w.kept, w.counts + 1, (int)m, st));
  } else {
    GU_CHECK(cudaMemsetAsync(w.counts + 1, 0, sizeof(int), st));
  }
  unsigned long long best = 0;
  int m2 = 0;
  GU_CHECK(cudaMemcpyAsync(&best, w.best, sizeof(best), cudaMemcpyDeviceToHost, st));
  GU_CHECK(cudaMemcpyAsync(&m2, w.counts + 1, sizeof(int), cudaMemcpyDeviceToHost, st));
  GU_CHECK(cudaStreamSynchronize(st));
  host_out[0] = ncomp;
  host_out[1] = (int64_t)(best >> 32);
  host_out[2] = m2;
  return GU_OK;
}

// phase 2: old id of each kept vertex (int32 n2), the champion's edges
// (int64 (m2, 2)) and CSR
extern "C" int gu_lcc_build(int64_t n, int64_t m, int64_t n2, int64_t m2, int32_t* out_old_ids,
                            int64_t* out_edges, int64_t* out_indptr, int32_t* out_indices,
                            void* workspace, size_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!workspace || ws_bytes < gu_lcc_workspace_size(n, m) || n2 < 1) {
    set_error("gu_lcc_build: bad arguments");
    return GU_ERR_ARG;
  }
  LccWs w = lcc_ws(n, m, (char*)workspace);
  ig_kept_ids<<<IG_BLOCKS, IG_THREADS, 0, st>>>((int)n, w.keep, w.remap, out_old_ids);
  GU_CHECK_LAUNCH("ig_kept_ids");
  return keys_to_graph(n2, m2, w.kept, w.both, w.both_sorted, w.deg, (long long*)out_edges,
                       (long long*)out_indptr,
                       out_indices, w.tmp, w.tmp_bytes, st);
}
