// order.cu -- a locality relabelling of the symmetrised kNN graph for the
// SGD epochs (csrc/sgd.cu), and the graph re-expressed in the new ids.
//
// Hogwild SGD is statistical (D7 in SURVEY.md section 9): which ids the
// vertices carry inside the epochs does not change the algorithm, and the
// caller's coordinates and visit log are mapped back at the boundary.  A
// breadth-first order makes every vertex's neighbours carry nearby ids on
// geometric graphs (c5: a kNN graph of points in the plane), so the head's
// neighbour ids fit a narrow [min, max] window that travels in its edge
// record: a uniform negative candidate falls outside it with probability
// ~1 - width / n, and that two-compare test replaces most Bloom-word work.
//
// Order: levels of a BFS from a pseudo-peripheral vertex (a BFS from vertex
// 0, then a second one from the smallest id of its last level), vertices
// sorted by (level, id); vertices the second BFS does not reach follow in id
// order.  Levels are deterministic whatever order the atomics land in, and
// so is the sort: the relabelling is a pure function of the graph.
// The BFS runs as one cooperative kernel, a grid-wide barrier per level.
#include <climits>

#include <cooperative_groups.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <cstdlib>

#include "common.cuh"
#include "gumap.h"

namespace cg = cooperative_groups;

namespace gu {
namespace {

constexpr int ORD_THREADS = 256;

__global__ void bfs_init(int n, int* __restrict__ level, int* __restrict__ cnt, int cnt_len,
                         int root, int* __restrict__ q0) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    level[i] = i == root ? 0 : -1;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt_len; i += gridDim.x * blockDim.x)
    cnt[i] = i == 0 ? 1 : 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) q0[0] = root;
}

// level-synchronous BFS: frontier of level l in q[l & 1] (cnt[l] entries);
// a vertex joins level l + 1 when its CAS from -1 succeeds.  On exit
// out[0] = last non-empty level, out[1] = its smallest vertex id.
#ifndef ORD_GRID_PER_SM
#define ORD_GRID_PER_SM 2
#endif
__global__ void __launch_bounds__(ORD_THREADS)
    bfs_levels_coop(int n, const int* __restrict__ indptr, const int* __restrict__ indices,
                    int* __restrict__ level, int* __restrict__ cnt, int* __restrict__ q0,
                    int* __restrict__ q1, int* __restrict__ out) {
  cg::grid_group grid = cg::this_grid();
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nthr = (long long)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  int l = 0;
  for (;;) {
    const int fsize = *(volatile int*)&cnt[l];
    int* cur = (l & 1) ? q1 : q0;
    int* nxt = (l & 1) ? q0 : q1;
    // one warp per frontier vertex, its lanes over the adjacency: a level of
    // a deep BFS (c5's kNN graph: ~1,400 levels of a few thousand vertices) is
    // then a couple of memory round trips instead of deg(u) dependent atomics;
    // visited neighbours are skipped by an L2 read before the CAS
    for (long long i = tid >> 5; i < fsize; i += nthr >> 5) {
      const int u = cur[i];
      const int b = __ldg(indptr + u), e = __ldg(indptr + u + 1);
      for (int p = b + lane; p < e; p += 32) {
        const int w = __ldg(indices + p);
        if (__ldcg(&level[w]) == -1 && atomicCAS(&level[w], -1, l + 1) == -1)
          nxt[atomicAdd(&cnt[l + 1], 1)] = w;
      }
    }
    grid.sync();
    if (*(volatile int*)&cnt[l + 1] == 0) break;
    l++;
  }
  // the last level sits in q[l & 1]: its smallest id
  if (blockIdx.x == 0) {
    __shared__ int smin[ORD_THREADS / 32];
    const int* last = (l & 1) ? q1 : q0;
    const int fsize = cnt[l];
    int m = INT_MAX;
    for (int i = threadIdx.x; i < fsize; i += blockDim.x) m = min(m, last[i]);
    for (int o = 16; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) smin[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int k = 1; k < ORD_THREADS / 32; k++) m = min(m, smin[k]);
      out[0] = l;
      out[1] = min(m, smin[0]);
    }
  }
}

__global__ void level_keys(int n, const int* __restrict__ level,
                           unsigned long long* __restrict__ keys) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const unsigned lv = level[i] < 0 ? 0x7fffffffu : (unsigned)level[i];
    keys[i] = ((unsigned long long)lv << 32) | (unsigned)i;
  }
}

// order[new] = old (low half of the sorted keys), perm[old] = new
__global__ void keys_to_perm(int n, const unsigned long long* __restrict__ keys,
                             int* __restrict__ order, int* __restrict__ perm) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int old = (int)(unsigned)(keys[i] & 0xffffffffu);
    order[i] = old;
    perm[old] = i;
  }
}

// new-id adjacency: key (perm[u] << 32 | perm[w]) per entry; degrees in new order
__global__ void relabel_keys(int n, const int* __restrict__ indptr, const int* __restrict__ indices,
                             const int* __restrict__ perm, unsigned long long* __restrict__ keys,
                             int* __restrict__ newdeg) {
  const int lane = threadIdx.x & 31;
  for (long long w0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w0 < n;
       w0 += ((long long)gridDim.x * blockDim.x) >> 5) {
    const int u = (int)w0;
    const int b = __ldg(indptr + u), e = __ldg(indptr + u + 1);
    const unsigned long long hi = (unsigned long long)(unsigned)perm[u] << 32;
    for (int p = b + lane; p < e; p += 32) keys[p] = hi | (unsigned)perm[__ldg(indices + p)];
    if (lane == 0) newdeg[perm[u]] = e - b;
  }
}

__global__ void keys_low(long long m, const unsigned long long* __restrict__ keys,
                         int* __restrict__ out) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = (int)(unsigned)(keys[i] & 0xffffffffu);
}

unsigned blocks_for(long long items) {
  long long b = (items + ORD_THREADS - 1) / ORD_THREADS;
  if (b > 148LL * 8) b = 148LL * 8;
  return (unsigned)(b < 1 ? 1 : b);
}

struct OrdWs {
  int* level;
  int* cnt;
  int* q0;
  int* q1;
  int* out;
  unsigned long long* k0;
  unsigned long long* k1;
  int* newdeg;
  void* cub_tmp;
  size_t cub_bytes;
};

size_t ord_layout(long long n, long long m, char* base, OrdWs* ws) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = (off + bytes + 255) & ~(size_t)255;
    return o;
  };
  const long long kn = n > m ? n : m;
  size_t cub_bytes = 0, c2 = 0, c3 = 0;
  cub::DeviceRadixSort::SortKeys((void*)nullptr, cub_bytes, (unsigned long long*)nullptr,
                                 (unsigned long long*)nullptr, (int)kn);
  cub::DeviceScan::ExclusiveSum((void*)nullptr, c2, (int*)nullptr, (int*)nullptr, (int)(n + 1));
  if (c2 > cub_bytes) cub_bytes = c2;
  (void)c3;
  const size_t ol = take(4 * (size_t)n), oc = take(4 * (size_t)(n + 2)),
               oq0 = take(4 * (size_t)n + 4), oq1 = take(4 * (size_t)n + 4), oo = take(16),
               ok0 = take(8 * (size_t)kn), ok1 = take(8 * (size_t)kn),
               od = take(4 * (size_t)(n + 1)), ot = take(cub_bytes);
  if (base && ws) {
    ws->level = (int*)(base + ol);
    ws->cnt = (int*)(base + oc);
    ws->q0 = (int*)(base + oq0);
    ws->q1 = (int*)(base + oq1);
    ws->out = (int*)(base + oo);
    ws->k0 = (unsigned long long*)(base + ok0);
    ws->k1 = (unsigned long long*)(base + ok1);
    ws->newdeg = (int*)(base + od);
    ws->cub_tmp = base + ot;
    ws->cub_bytes = cub_bytes;
  }
  return off;
}

int run_bfs(int n, const int* indptr, const int* indices, int root, const OrdWs& ws,
            cudaStream_t st) {
  bfs_init<<<blocks_for(n + 2), ORD_THREADS, 0, st>>>(n, ws.level, ws.cnt, n + 2, root, ws.q0);
  GU_CHECK_LAUNCH("bfs_init");
  int dev = 0, sms = 0, per_sm = 0;
  GU_CHECK(cudaGetDevice(&dev));
  GU_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  GU_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bfs_levels_coop, ORD_THREADS, 0));
  if (per_sm < 1) per_sm = 1;
  // CTAs per SM: a grid barrier per BFS level costs more the more CTAs join it
  // (GU_ORD_GRID_PER_SM, default below)
  static const int want = [] {
    const char* v = getenv("GU_ORD_GRID_PER_SM");
    const int x = v ? atoi(v) : 0;
    return x >= 1 ? x : ORD_GRID_PER_SM;
  }();
  const unsigned grid = (unsigned)(sms * (per_sm < want ? per_sm : want));
  const int* ip = indptr;
  const int* ix = indices;
  int* lv = ws.level;
  int* cnt = ws.cnt;
  int* q0 = ws.q0;
  int* q1 = ws.q1;
  int* out = ws.out;
  void* args[] = {(void*)&n, (void*)&ip, (void*)&ix, (void*)&lv, (void*)&cnt, (void*)&q0,
                  (void*)&q1, (void*)&out};
  GU_CHECK(cudaLaunchCooperativeKernel((const void*)bfs_levels_coop, dim3(grid),
                                       dim3(ORD_THREADS), args, 0, st));
  return GU_OK;
}

}  // namespace
}  // namespace gu

using namespace gu;

extern "C" size_t gu_bfs_order_workspace_size(int64_t n, int64_t m) {
  return ord_layout(n, m, nullptr, nullptr);
}

extern "C" int gu_bfs_order(int64_t n, const int32_t* indptr, const int32_t* indices,
                            int32_t* order, int32_t* perm, int32_t* new_indptr,
                            int32_t* new_indices, int32_t* host_levels, void* workspace,
                            size_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 1 || n >= INT_MAX) {
    set_error("gu_bfs_order: bad n=%lld", (long long)n);
    return GU_ERR_ARG;
  }
  long long m = 0;
  GU_CHECK(cudaMemcpyAsync(&m, indptr + n, sizeof(int), cudaMemcpyDeviceToHost, st));
  GU_CHECK(cudaStreamSynchronize(st));
  m = (long long)(int)m;
  OrdWs ws;
  if (!workspace || ws_bytes < ord_layout(n, m, (char*)workspace, &ws)) {
    set_error("gu_bfs_order: workspace too small");
    return GU_ERR_WORKSPACE;
  }
  const int N = (int)n;
  // sweep 1 from vertex 0, sweep 2 from the smallest id of sweep 1's last level
  int rc = run_bfs(N, indptr, indices, 0, ws, st);
  if (rc) return rc;
  int res[2] = {0, 0};
  GU_CHECK(cudaMemcpyAsync(res, ws.out, sizeof(res), cudaMemcpyDeviceToHost, st));
  GU_CHECK(cudaStreamSynchronize(st));
  rc = run_bfs(N, indptr, indices, res[1], ws, st);
  if (rc) return rc;
  int res2[2] = {0, 0};
  GU_CHECK(cudaMemcpyAsync(res2, ws.out, sizeof(res2), cudaMemcpyDeviceToHost, st));
  // sort by (level, id)
  level_keys<<<blocks_for(n), ORD_THREADS, 0, st>>>(N, ws.level, ws.k0);
  GU_CHECK_LAUNCH("level_keys");
  size_t cb = ws.cub_bytes;
  int lv_bits = 1;
  while (lv_bits < 31 && (1LL << lv_bits) <= (long long)n) lv_bits++;
  cub::DoubleBuffer<unsigned long long> kb(ws.k0, ws.k1);
  GU_CHECK(cub::DeviceRadixSort::SortKeys(ws.cub_tmp, cb, kb, N, 0, 32 + 31, st));
  keys_to_perm<<<blocks_for(n), ORD_THREADS, 0, st>>>(N, kb.Current(), order, perm);
  GU_CHECK_LAUNCH("keys_to_perm");
  // the graph in new ids: rows sorted by new neighbour id
  if (new_indptr && new_indices && m > 0) {
    relabel_keys<<<blocks_for(n * 32LL), ORD_THREADS, 0, st>>>(N, indptr, indices, perm, ws.k0,
                                                              ws.newdeg);
    GU_CHECK_LAUNCH("relabel_keys");
    cub::DoubleBuffer<unsigned long long> eb(ws.k0, ws.k1);
    int hi_bits = lv_bits;
    cb = ws.cub_bytes;
    GU_CHECK(cub::DeviceRadixSort::SortKeys(ws.cub_tmp, cb, eb, (int)m, 0, 32 + hi_bits, st));
    keys_low<<<blocks_for(m), ORD_THREADS, 0, st>>>(m, eb.Current(), new_indices);
    GU_CHECK_LAUNCH("keys_low");
    GU_CHECK(cudaMemsetAsync(ws.newdeg + n, 0, sizeof(int), st));
    cb = ws.cub_bytes;
    GU_CHECK(cub::DeviceScan::ExclusiveSum(ws.cub_tmp, cb, ws.newdeg, new_indptr, N + 1, st));
  }
  GU_CHECK(cudaStreamSynchronize(st));
  if (host_levels) {
    host_levels[0] = res[0];
    host_levels[1] = res2[0];
  }
  return GU_OK;
}
