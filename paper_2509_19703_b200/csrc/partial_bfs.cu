// partial_bfs.cu -- K3: truncated multi-source BFS fused with kNN selection.
//
// Replaces the reference's partial_bfs_all (numba), /root/reference/pkg/src/
// graph_umap/_kernels.py:60-131, called from neighbors.py:137-180.  Output is
// bit-identical: the k hop-nearest others of every source, the level that
// crosses the budget subsampled by the reference's splitmix64 partial
// Fisher-Yates (state seed + gamma*(s+1)), rows sorted by (dist, id).
//
// The Fisher-Yates indexes the crossing level in the reference's FIFO
// *discovery order*.  A level-synchronous warp reproduces it without a queue:
// level L+1 in discovery order == its vertices sorted by (min rank of a parent
// in level L, vertex id).  Each warp expands a whole level
// at once (flattened adjacency of the frontier, 32 entries per step), inserts
// the neighbours into a shared-memory hash keyed by vertex id whose value is
// atomicMin((level << 20) | parent_rank), then sorts the new level by
// (rank, id) with a warp bitonic sort.
//
// Tiers (no host sync between them; counts live in device memory):
//   tier 1a  shared hash, CAP=128 discovered vertices per source, 8 warps/CTA
//   tier 1b  shared hash, CAP=1024 (sources that overflowed 1a)
//   tier 2   per-warp global stamp array of n ints, parents expanded
//            sequentially in queue order (any level size, any k)
#include <climits>
#include <cstdio>

#include "common.cuh"
#include "gumap.h"

namespace gu {
namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ unsigned hash_id(int w) { return (unsigned)w * 0x9E3779B1u; }

// warp bitonic sort of P (power of two, >= 32) 64-bit keys in shared memory
__device__ __forceinline__ void warp_bitonic_sort(long long* key, int P) {
  const int lane = lane_id();
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = lane; t < (P >> 1); t += 32) {
        int i = 2 * t - (t & (stride - 1));
        int j = i + stride;
        bool up = (i & size) == 0;
        long long a = key[i], b = key[j];
        if ((a > b) == up) {
          key[i] = b;
          key[j] = a;
        }
      }
      __syncwarp();
    }
  }
}

// Sort `count` (<= 32) entries held one per lane by (dist, id) and store.
__device__ __forceinline__ void store_sorted_row(int count, int my_v, int my_d,
                                                 int* out_nbr, int* out_dist) {
  const int lane = lane_id();
  int pos = 0;
  for (int j = 0; j < count; j++) {
    int vj = __shfl_sync(FULL, my_v, j);
    int dj = __shfl_sync(FULL, my_d, j);
    if (dj < my_d || (dj == my_d && vj < my_v)) pos++;
  }
  if (lane < count) {
    out_nbr[pos] = my_v;
    out_dist[pos] = my_d;
  }
}

template <int CAP>
struct Tier1 {
  static constexpr int HC = 2 * CAP;
  // per-warp shared layout (ints): disc[CAP] stage[CAP] key64[CAP](=2*CAP ints)
  //                                hkey[HC] hval[HC]
  // pre/beg of the frontier alias the key64 region (used before the sort).
  static constexpr int WORDS = CAP + CAP + 2 * CAP + 2 * HC + 4;
  static constexpr size_t BYTES = WORDS * sizeof(int);
};

template <int CAP, int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
    pbfs_tier1(const int* __restrict__ indptr, const int* __restrict__ indices,
               int K, unsigned long long seed, long long src_begin, long long nsrc,
               const int* __restrict__ list, const int* __restrict__ list_count,
               int* __restrict__ out_nbr, int* __restrict__ out_dist,
               int* __restrict__ out_cnt, int* __restrict__ ovf_list,
               int* __restrict__ ovf_count, unsigned long long* __restrict__ work) {
  constexpr int HC = Tier1<CAP>::HC;
  extern __shared__ __align__(16) int smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int* base = smem + warp * Tier1<CAP>::WORDS;
  int* disc = base;
  int* stage = disc + CAP;
  long long* key64 = reinterpret_cast<long long*>(stage + CAP);  // 2*CAP ints
  int* pre = reinterpret_cast<int*>(key64);                       // CAP+1 ints
  int* beg = pre + CAP + 1;                                       // CAP-1 .. ints
  int* hkey = stage + 3 * CAP;
  int* hval = hkey + HC;

  unsigned long long w_scanned = 0, w_expanded = 0;
  const long long total = list ? (long long)(*list_count) : nsrc;
  for (long long item = (long long)blockIdx.x * WARPS + warp; item < total;
       item += (long long)gridDim.x * WARPS) {
    const int s = list ? list[item] : (int)(src_begin + item);
    for (int i = lane; i < HC; i += 32) {
      hkey[i] = -1;
      hval[i] = INT_MAX;
    }
    __syncwarp();
    if (lane == 0) {
      unsigned h = hash_id(s) & (HC - 1);
      hkey[h] = s;
      hval[h] = 0;
      disc[0] = s;
    }
    __syncwarp();
    int lb = 0, le = 1, count = 0, depth = 0;
    bool ovf = false;
    int my_v = 0, my_d = 0;
    unsigned long long scanned = 0, expanded = 0;
    while (count < K) {
      const int f = le - lb;
      // ---- frontier degrees, exclusive prefix (pre), adjacency starts (beg)
      // beg aliases pre[CAP+1..]; frontier sizes f <= CAP-1 keep them apart.
      int carry = 0;
      for (int i0 = 0; i0 < f; i0 += 32) {
        int i = i0 + lane, d = 0, b = 0;
        if (i < f) {
          int u = disc[lb + i];
          b = __ldg(indptr + u);
          d = __ldg(indptr + u + 1) - b;
        }
        int inc = warp_incl_scan(d);
        if (i < f) {
          pre[i] = carry + inc - d;
          beg[i] = b;
        }
        carry += __shfl_sync(FULL, inc, 31);
      }
      __syncwarp();
      const int T = carry;
      scanned += T;
      expanded += f;
      depth++;
      const int tag = depth << 20;
      // ---- expand: flattened adjacency of the frontier, 32 entries per step
      int nst = 0;
      bool fail = false;
      for (int t0 = 0; t0 < T; t0 += 32) {
        const int t = t0 + lane;
        bool isnew = false;
        int w = -1;
        if (t < T) {
          int lo = 0, hi = f - 1;  // largest p with pre[p] <= t
          while (lo < hi) {
            int mid = (lo + hi + 1) >> 1;
            if (pre[mid] <= t) lo = mid; else hi = mid - 1;
          }
          w = __ldg(indices + beg[lo] + (t - pre[lo]));
          unsigned h = hash_id(w) & (HC - 1);
          int probe = 0;
          for (; probe < HC; probe++) {
            int old = atomicCAS(&hkey[h], -1, w);
            if (old == -1) {
              isnew = true;
              break;
            }
            if (old == w) break;
            h = (h + 1) & (HC - 1);
          }
          if (probe == HC) fail = true;
          else atomicMin(&hval[h], tag | lo);
        }
        unsigned bal = __ballot_sync(FULL, isnew);
        if (isnew) {
          int pos = nst + __popc(bal & lanemask_lt());
          if (pos < CAP) stage[pos] = w;
        }
        nst += __popc(bal);
      }
      __syncwarp();
      if (__any_sync(FULL, fail) || le + nst > CAP - 1) {
        ovf = true;
        break;
      }
      if (nst == 0) break;  // component exhausted
      // ---- order the new level by (min parent rank, id) == discovery order
      int P = 32;
      while (P < nst) P <<= 1;
      for (int i = lane; i < P; i += 32) {
        long long key = LLONG_MAX;
        if (i < nst) {
          int w = stage[i];
          unsigned h = hash_id(w) & (HC - 1);
          while (hkey[h] != w) h = (h + 1) & (HC - 1);
          key = ((long long)(hval[h] & 0xFFFFF) << 32) | (unsigned)w;
        }
        key64[i] = key;
      }
      __syncwarp();
      warp_bitonic_sort(key64, P);
      for (int i = lane; i < nst; i += 32) disc[le + i] = (int)(key64[i] & 0xffffffffLL);
      __syncwarp();
      const int remaining = K - count;
      int take = nst;
      if (nst > remaining) {
        // random subset of the crossing level (_kernels.py:98-105)
        if (lane == 0) {
          unsigned long long st = seed + SPLIT_GAMMA * (unsigned long long)(s + 1);
          for (int i = 0; i < remaining; i++) {
            int j = i + (int)(splitmix_next(st) % (unsigned long long)(nst - i));
            int a = disc[le + i];
            disc[le + i] = disc[le + j];
            disc[le + j] = a;
          }
        }
        __syncwarp();
        take = remaining;
      }
      if (lane >= count && lane < count + take) {
        my_v = disc[le + lane - count];
        my_d = depth;
      }
      count += take;
      lb = le;
      le += nst;
    }
    if (ovf) {
      if (lane == 0) ovf_list[atomicAdd(ovf_count, 1)] = s;
      continue;
    }
    const long long row = (long long)s - src_begin;
    store_sorted_row(count, my_v, my_d, out_nbr + row * K, out_dist + row * K);
    if (lane == 0) out_cnt[row] = count;
    w_scanned += scanned;
    w_expanded += expanded;
  }
  if (work && lane == 0) {
    atomicAdd(work, w_scanned);
    atomicAdd(work + 1, w_expanded);
  }
}

// ----------------------------------------------------------------- tier 2
// Exact FIFO emulation: parents in queue order, each parent's sorted
// adjacency in 32-entry chunks; per-warp stamp array (value s+1) of n ints.
__global__ void __launch_bounds__(256)
    pbfs_tier2(int n, const int* __restrict__ indptr, const int* __restrict__ indices,
               int K, unsigned long long seed, long long src_begin,
               const int* __restrict__ list, const int* __restrict__ list_count,
               int* __restrict__ slots, int nslots, int* __restrict__ out_nbr,
               int* __restrict__ out_dist, int* __restrict__ out_cnt,
               unsigned long long* __restrict__ work) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (gw >= nslots) return;
  int* stamp = slots + (size_t)gw * 2 * (size_t)n;
  int* disc = stamp + n;
  const int total = *list_count;
  unsigned long long w_scanned = 0, w_expanded = 0;
  for (int item = gw; item < total; item += nslots) {
    const int s = list[item];
    const int mark = s + 1;
    if (lane == 0) {
      stamp[s] = mark;
      disc[0] = s;
    }
    __syncwarp();
    int lb = 0, le = 1, count = 0, depth = 0;
    while (count < K) {
      int nst = 0;
      for (int p = lb; p < le; p++) {
        const int u = disc[p];
        const int b = __ldg(indptr + u), e = __ldg(indptr + u + 1);
        w_scanned += (e - b);
        w_expanded += 1;
        for (int off = b; off < e; off += 32) {
          const int idx = off + lane;
          int w = -1;
          bool isnew = false;
          if (idx < e) {
            w = __ldg(indices + idx);
            isnew = stamp[w] != mark;
          }
          unsigned bal = __ballot_sync(FULL, isnew);
          if (isnew) {
            stamp[w] = mark;
            disc[le + nst + __popc(bal & lanemask_lt())] = w;
          }
          nst += __popc(bal);
          __syncwarp();
        }
      }
      depth++;
      if (nst == 0) break;
      const int remaining = K - count;
      int take = nst;
      if (nst > remaining) {
        if (lane == 0) {
          unsigned long long st = seed + SPLIT_GAMMA * (unsigned long long)(s + 1);
          for (int i = 0; i < remaining; i++) {
            int j = i + (int)(splitmix_next(st) % (unsigned long long)(nst - i));
            int a = disc[le + i];
            disc[le + i] = disc[le + j];
            disc[le + j] = a;
          }
        }
        __syncwarp();
        take = remaining;
      }
      // output entries count..count+take: the first `take` of this level
      const long long row = (long long)s - src_begin;
      for (int i = lane; i < take; i += 32) {
        out_nbr[row * K + count + i] = disc[le + i];
        out_dist[row * K + count + i] = depth;
      }
      count += take;
      lb = le;
      le += nst;
    }
    __syncwarp();
    // sort the row by (dist, id): entries come level by level, so only ids
    // inside each level block need ordering (insertion sort, lane 0)
    const long long row = (long long)s - src_begin;
    if (lane == 0) {
      int* rn = out_nbr + row * K;
      int* rd = out_dist + row * K;
      for (int i = 1; i < count; i++) {
        int a = rn[i], d = rd[i], j = i - 1;
        while (j >= 0 && (rd[j] > d || (rd[j] == d && rn[j] > a))) {
          rn[j + 1] = rn[j];
          rd[j + 1] = rd[j];
          j--;
        }
        rn[j + 1] = a;
        rd[j + 1] = d;
      }
      out_cnt[row] = count;
    }
    __syncwarp();
  }
  if (work && lane == 0) {
    atomicAdd(work, w_scanned);
    atomicAdd(work + 1, w_expanded);
  }
}

__global__ void fill_range_list(int* list, int* count, long long src_begin, long long nsrc) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nsrc) list[i] = (int)(src_begin + i);
  if (i == 0) *count = (int)nsrc;
}

__global__ void clear_slots_if_needed(int* slots, size_t words, const int* count) {
  if (*count == 0) return;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < words;
       i += (size_t)gridDim.x * blockDim.x)
    slots[i] = 0;
}

constexpr int T1A_CAP = 128, T1A_WARPS = 8;
constexpr int T1B_CAP = 1024, T1B_WARPS = 2;

struct PbfsWs {
  int* ovfA;
  int* ovfB;
  int* counts;  // [0]=ovfA count, [1]=ovfB count
  unsigned long long* work;
  int* slots;
};

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

size_t pbfs_ws_layout(long long n, long long nsrc, int slots, char* base, PbfsWs* ws) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align256(off + bytes);
    return o;
  };
  size_t oA = take(sizeof(int) * (size_t)(nsrc + 1));
  size_t oB = take(sizeof(int) * (size_t)(nsrc + 1));
  size_t oC = take(sizeof(int) * 4);
  size_t oW = take(sizeof(unsigned long long) * 2);
  size_t oS = take(sizeof(int) * 2 * (size_t)n * (size_t)slots);
  if (ws && base) {
    ws->ovfA = (int*)(base + oA);
    ws->ovfB = (int*)(base + oB);
    ws->counts = (int*)(base + oC);
    ws->work = (unsigned long long*)(base + oW);
    ws->slots = (int*)(base + oS);
  }
  return off;
}

int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

}  // namespace
}  // namespace gu

using namespace gu;

extern "C" size_t gu_partial_bfs_workspace_size(int64_t n, int64_t nsrc, int32_t tier2_warps) {
  return pbfs_ws_layout(n, nsrc, tier2_warps > 0 ? tier2_warps : 1, nullptr, nullptr);
}

extern "C" int gu_partial_bfs_knn(int64_t n, const int32_t* indptr, const int32_t* indices,
                                  int32_t k, uint64_t seed, int64_t src_begin, int64_t src_end,
                                  int32_t* out_nbr, int32_t* out_dist, int32_t* out_count,
                                  uint64_t* work_counters, void* workspace, size_t ws_bytes,
                                  int32_t tier2_warps, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const long long nsrc = src_end - src_begin;
  if (n < 0 || n >= INT_MAX || k < 0 || src_begin < 0 || src_end > n || nsrc < 0) {
    set_error("gu_partial_bfs_knn: bad arguments (n=%lld k=%d range=[%lld,%lld))",
              (long long)n, k, (long long)src_begin, (long long)src_end);
    return GU_ERR_ARG;
  }
  if (nsrc == 0) return GU_OK;
  if (tier2_warps < 1) tier2_warps = 1;
  PbfsWs ws;
  size_t need = pbfs_ws_layout(n, nsrc, tier2_warps, (char*)workspace, &ws);
  if (!workspace || ws_bytes < need) {
    set_error("gu_partial_bfs_knn: workspace %zu < %zu bytes", ws_bytes, need);
    return GU_ERR_WORKSPACE;
  }
  unsigned long long* work = (unsigned long long*)work_counters;
  if (work) GU_CHECK(cudaMemsetAsync(work, 0, 2 * sizeof(unsigned long long), st));
  GU_CHECK(cudaMemsetAsync(ws.counts, 0, 4 * sizeof(int), st));
  if (k == 0) {
    GU_CHECK(cudaMemsetAsync(out_count, 0, sizeof(int32_t) * nsrc, st));
    return GU_OK;
  }
  const int sms = sm_count();
  if (k <= 32) {
    {
      constexpr size_t smem = Tier1<T1A_CAP>::BYTES * T1A_WARPS;
      auto kern = pbfs_tier1<T1A_CAP, T1A_WARPS>;
      GU_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      int per_sm = 0;
      GU_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T1A_WARPS * 32, smem));
      long long blocks = (nsrc + T1A_WARPS - 1) / T1A_WARPS;
      long long cap = (long long)sms * (per_sm > 0 ? per_sm : 1) * 8;
      if (blocks > cap) blocks = cap;
      kern<<<(unsigned)blocks, T1A_WARPS * 32, smem, st>>>(
          indptr, indices, k, seed, src_begin, nsrc, nullptr, nullptr, out_nbr, out_dist,
          out_count, ws.ovfA, ws.counts + 0, work);
      GU_CHECK_LAUNCH("pbfs_tier1<128>");
    }
    {
      constexpr size_t smem = Tier1<T1B_CAP>::BYTES * T1B_WARPS;
      auto kern = pbfs_tier1<T1B_CAP, T1B_WARPS>;
      GU_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      int per_sm = 0;
      GU_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T1B_WARPS * 32, smem));
      long long blocks = (long long)sms * (per_sm > 0 ? per_sm : 1);
      kern<<<(unsigned)blocks, T1B_WARPS * 32, smem, st>>>(
          indptr, indices, k, seed, src_begin, nsrc, ws.ovfA, ws.counts + 0, out_nbr, out_dist,
          out_count, ws.ovfB, ws.counts + 1, work);
      GU_CHECK_LAUNCH("pbfs_tier1<1024>");
    }
  } else {
    // k > 32: every source goes straight to the exact tier-2 path
    fill_range_list<<<(unsigned)((nsrc + 255) / 256), 256, 0, st>>>(ws.ovfB, ws.counts + 1,
                                                                   src_begin, nsrc);
    GU_CHECK_LAUNCH("fill_range_list");
  }
  {
    size_t words = (size_t)2 * (size_t)n * (size_t)tier2_warps;
    clear_slots_if_needed<<<(unsigned)(sms * 4), 256, 0, st>>>(ws.slots, words, ws.counts + 1);
    GU_CHECK_LAUNCH("clear_slots_if_needed");
    unsigned blocks = (unsigned)((tier2_warps * 32 + 255) / 256);
    pbfs_tier2<<<blocks, 256, 0, st>>>((int)n, indptr, indices, k, seed, src_begin, ws.ovfB,
                                       ws.counts + 1, ws.slots, tier2_warps, out_nbr, out_dist,
                                       out_count, work);
    GU_CHECK_LAUNCH("pbfs_tier2");
  }
  return GU_OK;
}

extern "C" int gu_partial_bfs_overflow_counts(void* workspace, int64_t nsrc, int32_t* host_out2) {
  PbfsWs ws;
  pbfs_ws_layout(1, nsrc, 1, (char*)workspace, &ws);
  GU_CHECK(cudaMemcpy(host_out2, ws.counts, 2 * sizeof(int), cudaMemcpyDeviceToHost));
  return GU_OK;
}
