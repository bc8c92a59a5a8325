// full_bfs.cu -- K2: 64-source bitset BFS (all_pairs_bfs) and the fused
// full-BFS kNN with the reference's numpy tie-break.
//
// Replaces:
//   apsp_rows               /root/reference/pkg/src/graph_umap/_kernels.py:33-57
//   all_pairs_bfs           neighbors.py:120-134
//   knn_from_full_distances neighbors.py:183-237 (PCG64 ties, neighbors.py:213-216)
//
// One CTA owns a batch of 64 sources (one bit each in a uint64 word per
// vertex) and runs the levels itself, persistent over batches:
//   level 1   push: each source's sorted adjacency ORs its bit into level[1]
//   level l   pull: new[v] = OR_{u in N(v)} level[l-1][u] & ~vis[v] & active
// Per-source level counts come from warp ballots; in kNN mode a source
// retires at the level where its running count reaches k (the k-th distance)
// or when its component is exhausted, and the batch stops when all 64 have
// retired -- the n x n matrix never exists.  Selection then reads the level
// words: levels < kth in (level, id) order, and the k-th distance ties by the
// reference's permutation: SeedSequence(seed, spawn_key=(v,)) -> PCG64 ->
// shuffle, picking the perm[0..need) -th tie in ascending id.
#include <climits>

#include "common.cuh"
#include "gumap.h"

namespace gu {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int FB_THREADS = 512;
constexpr int FB_WARPS = FB_THREADS / 32;

enum Mode { MODE_KNN = 0, MODE_APSP = 1, MODE_STRESS = 2 };

// MODE_STRESS (metrics.py:106-131 fused into the BFS): every (source, vertex)
// pair reached at level d adds its stress terms to per-thread float64 sums --
// the hop rows never exist.  pass2 = 0: (delta/d, delta^2/d^2) for the scale;
// pass2 = 1: (1 - delta*scale/d)^2.  acc[blockIdx.x] receives the CTA's sums
// (fixed ownership: deterministic); flag is set if a source misses vertices.
struct StressArgs {
  const double2* xy;
  const double* scale;
  double2* acc;
  int* flag;
  int pass2;
  const int* sources;  // nullable: BFS from sources[src_begin .. src_end) instead of the ids
};

struct FbShared {
  int cnt[64];
  int cum[64];
  int kth[64];
  int low[64];
  int tk[64];
  int lastlvl[64];
  unsigned keep[2];
  int anynew;  // MODE_APSP: a vertex was discovered in the level just finished
  unsigned long long active;
  double2 sxy[64];
  double red[2][FB_WARPS];
};

// scipy cdist (no contraction) and the stress terms of one pair at level d
__device__ __forceinline__ void stress_term(double2 p, double2 q, int lvl, const StressArgs& sa,
                                            double scale, double& a, double& b) {
  const double dx = __dsub_rn(p.x, q.x), dy = __dsub_rn(p.y, q.y);
  const double delta = __dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
  const double d = (double)lvl;
  if (!sa.pass2) {
    a = __dadd_rn(a, __ddiv_rn(delta, d));
    b = __dadd_rn(b, __ddiv_rn(__dmul_rn(delta, delta), __dmul_rn(d, d)));
  } else {
    const double u = __dsub_rn(1.0, __ddiv_rn(__dmul_rn(delta, scale), d));
    a = __dadd_rn(a, __dmul_rn(u, u));
  }
}

__device__ __forceinline__ void sort_small_ids(int* ids, int m) {
  // ascending sort of m ids in global/shared memory by one warp
  const int lane = lane_id();
  if (m <= 32) {
    int my = lane < m ? ids[lane] : INT_MAX;
    int pos = 0;
    for (int j = 0; j < m; j++) {
      int vj = __shfl_sync(FULL, my, j);
      if (vj < my) pos++;
    }
    __syncwarp();
    if (lane < m) ids[pos] = my;
    __syncwarp();
  } else {
    if (lane == 0) {
      for (int i = 1; i < m; i++) {
        int a = ids[i], j = i - 1;
        while (j >= 0 && ids[j] > a) {
          ids[j + 1] = ids[j];
          j--;
        }
        ids[j + 1] = a;
      }
    }
    __syncwarp();
  }
}

template <int MODE>
__global__ void __launch_bounds__(FB_THREADS)
    msbfs_kernel(int n, const int* __restrict__ indptr, const int* __restrict__ indices,
                 int K, unsigned long long seed, long long src_begin, long long src_end,
                 int* __restrict__ out_nbr, int* __restrict__ out_dist, int* __restrict__ out_cnt,
                 int* __restrict__ out_rows, char* __restrict__ ws, size_t slot_bytes, int L,
                 unsigned long long* __restrict__ work, StressArgs sa) {
  __shared__ FbShared sh;
  double st_a = 0.0, st_b = 0.0;
  const double st_scale = (MODE == MODE_STRESS && sa.pass2) ? *sa.scale : 1.0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned long long* vis = reinterpret_cast<unsigned long long*>(ws + blockIdx.x * slot_bytes);
  unsigned long long* stack = vis + n;
  int* perm_base = reinterpret_cast<int*>(stack + (size_t)L * n);
  const long long nsrc = src_end - src_begin;
  const long long nbatches = (nsrc + 63) / 64;
  unsigned long long te = 0, levels_run = 0;

  for (long long bi = blockIdx.x; bi < nbatches; bi += gridDim.x) {
    const long long s0 = src_begin + bi * 64;
    const int nb = (int)min(64LL, src_end - s0);
    auto level = [&](int l) -> unsigned long long* {
      return stack + (size_t)(MODE != MODE_KNN ? (l & 1) : l) * n;
    };
    unsigned long long* l1 = level(1);
    for (int v = tid; v < n; v += FB_THREADS) {
      vis[v] = 0ull;
      l1[v] = 0ull;
    }
    // APSP rows: every (source, vertex) entry is written exactly once -- 0 for
    // the source itself here, its level when it is discovered, GU_INF32 by
    // the unreached pass after the levels (no full-row initialisation pass)
    if (MODE == MODE_APSP && tid < nb) out_rows[(s0 - src_begin + tid) * (long long)n + s0 + tid] = 0;
    // source id of bit b: s0 + b, or the listed source in stress mode
    auto src_of = [&](int b) -> int {
      return (MODE == MODE_STRESS && sa.sources) ? sa.sources[s0 + b] : (int)(s0 + b);
    };
    if (MODE == MODE_STRESS && tid < nb) sh.sxy[tid] = sa.xy[src_of(tid)];
    if (tid < 64) {
      sh.cnt[tid] = 0;
      sh.cum[tid] = 0;
      sh.kth[tid] = -1;
      sh.low[tid] = 0;
      sh.tk[tid] = 0;
      sh.lastlvl[tid] = 0;
    }
    if (tid == 0) {
      sh.active = nb == 64 ? ~0ull : ((1ull << nb) - 1ull);
      sh.anynew = 0;
    }
    __syncthreads();
    // ---- level 0 / level 1 (push from the sources' sorted adjacency)
    for (int b = warp; b < nb; b += FB_WARPS) {
      const int s = src_of(b);
      const int beg = __ldg(indptr + s), end = __ldg(indptr + s + 1);
      if (lane == 0) {
        atomicOr(&vis[s], 1ull << b);
        sh.cnt[b] = end - beg;
        if (MODE == MODE_APSP && end > beg) sh.anynew = 1;
      }
      te += (lane == 0) ? (unsigned long long)(end - beg) : 0ull;
      int* row = MODE == MODE_APSP ? out_rows + (s0 - src_begin + b) * (long long)n : nullptr;
      for (int p = beg + lane; p < end; p += 32) {
        int w = __ldg(indices + p);
        atomicOr(&l1[w], 1ull << b);
        if (MODE == MODE_APSP) row[w] = 1;
        if (MODE == MODE_STRESS) stress_term(sh.sxy[b], sa.xy[w], 1, sa, st_scale, st_a, st_b);
      }
    }
    __syncthreads();
    int l = 1;
    for (;;) {
      // ---- retire sources whose running count reached K (kNN) or whose
      //      component is exhausted (both modes)
      if (tid < 64) {
        const int b = tid;
        bool act = (sh.active >> b) & 1ull;
        bool keep = act;
        if (MODE == MODE_APSP) {
          // no per-source counts in APSP mode: every source runs until a level
          // discovers nothing for any of them
          keep = act && sh.anynew != 0;
          sh.cnt[b] = 0;
          act = false;  // skip the count bookkeeping below
        }
        if (act) {
          int c = sh.cnt[b];
          if (c == 0) {
            keep = false;  // exhausted: everything reachable is in levels < l
          } else {
            sh.lastlvl[b] = l;
            if (MODE == MODE_KNN && sh.cum[b] + c >= K) {
              sh.kth[b] = l;
              sh.low[b] = sh.cum[b];
              sh.tk[b] = c;
              keep = false;
            }
            sh.cum[b] += c;
          }
          sh.cnt[b] = 0;
        }
        unsigned bal = __ballot_sync(FULL, keep);
        if (lane == 0) sh.keep[warp] = bal;
      }
      __syncthreads();
      if (tid == 0) sh.active = (unsigned long long)sh.keep[0] | ((unsigned long long)sh.keep[1] << 32);
      __syncthreads();
      const unsigned long long active = sh.active;
      if (active == 0ull) break;
      levels_run++;
      if (MODE == MODE_APSP && tid == 0) sh.anynew = 0;  // read by the retire step above
      // ---- fold the level just finished into vis
      {
        unsigned long long* prev = level(l);
        if (l == 1) {
          for (int v = tid; v < n; v += FB_THREADS) vis[v] |= prev[v];
        }
      }
      __syncthreads();
      const int nl = l + 1;
      unsigned long long* prev = level(l);
      unsigned long long* next = level(nl);
      int my_cnt0 = 0, my_cnt1 = 0;
      for (int v0 = warp * 32; v0 < n; v0 += FB_THREADS) {
        const int v = v0 + lane;
        unsigned long long nw = 0ull;
        if (v < n) {
          const unsigned long long vv = vis[v];
          const unsigned long long need = ~vv & active;
          if (need != 0ull) {
            const int beg = __ldg(indptr + v), end = __ldg(indptr + v + 1);
            unsigned long long acc = 0ull;
            int p = beg;
            // bottom-up early exit: stop once every source still looking for
            // v has found it (dense late levels touch a few neighbours); the
            // new bits are the same as with the full OR
            for (; p + 4 <= end; p += 4) {
              const int i0 = __ldg(indices + p), i1 = __ldg(indices + p + 1),
                        i2 = __ldg(indices + p + 2), i3 = __ldg(indices + p + 3);
              acc |= prev[i0] | prev[i1] | prev[i2] | prev[i3];
              if ((acc & need) == need) {
                p += 4;
                break;
              }
            }
            if ((acc & need) != need)
              for (; p < end; p++) acc |= prev[__ldg(indices + p)];
            te += (unsigned long long)(p - beg);  // entries actually read
            nw = acc & need;
            if (nw) vis[v] = vv | nw;
          }
          next[v] = nw;
        }
        unsigned long long any = nw;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) any |= __shfl_xor_sync(FULL, any, o);
        if (MODE == MODE_APSP) {
          // rows written coalesced, one source bit at a time; no counts
          if (any && lane == 0) sh.anynew = 1;
          while (any) {
            const int b = __ffsll((long long)any) - 1;
            any &= any - 1ull;
            if ((nw >> b) & 1ull) out_rows[(s0 - src_begin + b) * (long long)n + v] = nl;
          }
        }
        while (MODE != MODE_APSP && any) {
          const int b = __ffsll((long long)any) - 1;
          any &= any - 1ull;
          const int c = __popc(__ballot_sync(FULL, (nw >> b) & 1ull));
          if (lane == (b & 31)) {
            if (b < 32) my_cnt0 += c; else my_cnt1 += c;
          }
          if (MODE == MODE_APSP && ((nw >> b) & 1ull))
            out_rows[(s0 - src_begin + b) * (long long)n + v] = nl;
          if (MODE == MODE_STRESS && ((nw >> b) & 1ull))
            stress_term(sh.sxy[b], sa.xy[v], nl, sa, st_scale, st_a, st_b);
        }
      }
      if (my_cnt0) atomicAdd(&sh.cnt[lane], my_cnt0);
      if (my_cnt1) atomicAdd(&sh.cnt[lane + 32], my_cnt1);
      __syncthreads();
      l = nl;
      if (MODE == MODE_KNN && l >= L) break;  // unreachable by construction
    }
    if (MODE == MODE_STRESS && tid < nb && sh.cum[tid] + 1 < n) atomicOr(sa.flag, 1);
    if (MODE == MODE_APSP) {
      // unreached (source, vertex) pairs: GU_INF32 (none on a connected graph)
      const unsigned long long mine = nb == 64 ? ~0ull : ((1ull << nb) - 1ull);
      for (int v = tid; v < n; v += FB_THREADS) {
        unsigned long long miss = ~vis[v] & mine;
        while (miss) {
          const int b = __ffsll((long long)miss) - 1;
          miss &= miss - 1ull;
          if (v != (int)(s0 + b)) out_rows[(s0 - src_begin + b) * (long long)n + v] = GU_INF32;
        }
      }
    }
    if (MODE == MODE_KNN) {
      // ---- selection, one warp per source
      int* perm = perm_base + (size_t)warp * n;
      for (int b = warp; b < nb; b += FB_WARPS) {
        const int s = (int)(s0 + b);
        const long long row = s0 - src_begin + b;
        int* rn = out_nbr + row * K;
        int* rd = out_dist + row * K;
        const int kth = sh.kth[b];
        const int lastfull = kth >= 0 ? kth - 1 : sh.lastlvl[b];
        const int sbeg = __ldg(indptr + s), send = __ldg(indptr + s + 1);
        int pos = 0;
        // levels 1..lastfull: every vertex, (level, id) order
        for (int lv = 1; lv <= lastfull; lv++) {
          if (lv == 1) {
            for (int p = sbeg + lane; p < send; p += 32) {
              rn[pos + (p - sbeg)] = __ldg(indices + p);
              rd[pos + (p - sbeg)] = 1;
            }
            pos += send - sbeg;
          } else {
            const unsigned long long* lw = level(lv);
            for (int v0 = 0; v0 < n; v0 += 32) {
              const int v = v0 + lane;
              const bool bit = v < n && ((lw[v] >> b) & 1ull);
              const unsigned bal = __ballot_sync(FULL, bit);
              if (bit) {
                int q = pos + __popc(bal & lanemask_lt());
                rn[q] = v;
                rd[q] = lv;
              }
              pos += __popc(bal);
            }
          }
        }
        if (kth >= 0) {
          const int T = sh.tk[b];
          const int need = K - sh.low[b];
          if (need == T) {
            // every tie is picked: emit the whole level
            if (kth == 1) {
              for (int p = sbeg + lane; p < send; p += 32) {
                rn[pos + (p - sbeg)] = __ldg(indices + p);
                rd[pos + (p - sbeg)] = 1;
              }
            } else {
              const unsigned long long* lw = level(kth);
              int q0 = pos;
              for (int v0 = 0; v0 < n; v0 += 32) {
                const int v = v0 + lane;
                const bool bit = v < n && ((lw[v] >> b) & 1ull);
                const unsigned bal = __ballot_sync(FULL, bit);
                if (bit) {
                  int q = q0 + __popc(bal & lanemask_lt());
                  rn[q] = v;
                  rd[q] = kth;
                }
                q0 += __popc(bal);
              }
            }
          } else {
            // numpy: default_rng(SeedSequence(seed, spawn_key=(v,))).permutation(T)
            for (int i = lane; i < T; i += 32) perm[i] = i;
            __syncwarp();
            if (lane == 0) {
              Pcg64 rng;
              pcg64_from_seedseq(rng, seed, (unsigned long long)s);
              for (int i = T - 1; i >= 1; i--) {
                int j = (int)rng.interval((unsigned long long)i);
                int t = perm[i];
                perm[i] = perm[j];
                perm[j] = t;
              }
            }
            __syncwarp();
            // picked[q] = ties[perm[q]] (ties in ascending id)
            if (kth == 1) {
              for (int q = lane; q < need; q += 32) rn[pos + q] = __ldg(indices + sbeg + perm[q]);
            } else {
              const unsigned long long* lw = level(kth);
              int R = 0;
              for (int v0 = 0; v0 < n && R < T; v0 += 32) {
                const int v = v0 + lane;
                const bool bit = v < n && ((lw[v] >> b) & 1ull);
                const unsigned bal = __ballot_sync(FULL, bit);
                const int c = __popc(bal);
                if (c) {
                  for (int q = lane; q < need; q += 32) {
                    int r = perm[q];
                    if (r >= R && r < R + c) rn[pos + q] = v0 + (int)__fns(bal, 0, r - R + 1);
                  }
                }
                R += c;
              }
            }
            __syncwarp();
            for (int q = lane; q < need; q += 32) rd[pos + q] = kth;
            __syncwarp();
            sort_small_ids(rn + pos, need);
          }
          if (lane == 0) out_cnt[row] = K;
        } else {
          if (lane == 0) out_cnt[row] = pos;
        }
        __syncwarp();
      }
    }
    __syncthreads();
  }
  if (MODE == MODE_STRESS) {
    for (int o = 16; o > 0; o >>= 1) {
      st_a += __shfl_down_sync(FULL, st_a, o);
      st_b += __shfl_down_sync(FULL, st_b, o);
    }
    if (lane == 0) {
      sh.red[0][warp] = st_a;
      sh.red[1][warp] = st_b;
    }
    __syncthreads();
    if (tid == 0) {
      double x = 0.0, y = 0.0;
      for (int i = 0; i < FB_WARPS; i++) {
        x += sh.red[0][i];
        y += sh.red[1][i];
      }
      sa.acc[blockIdx.x] = make_double2(x, y);
    }
  }
  // TE is accumulated per thread; reduce per warp
  te = warp_sum(te);
  if (work && lane == 0) {
    atomicAdd(work, te);
    if (warp == 0) atomicAdd(work + 1, levels_run);
  }
}

// ------------------------------------------------ kNN from explicit rows
__global__ void __launch_bounds__(256)
    knn_rows_kernel(int n, const int* __restrict__ rows, long long row_begin, long long nrows,
                    int K, unsigned long long seed, int* __restrict__ out_nbr,
                    int* __restrict__ out_dist, int* __restrict__ out_cnt, int* __restrict__ scratch,
                    int nslots) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (gw >= nslots) return;
  int* ids = scratch + (size_t)gw * 2 * n;
  int* perm = ids + n;
  for (long long r = gw; r < nrows; r += nslots) {
    const int v = (int)(row_begin + r);
    const int* R = rows + r * (long long)n;
    int* rn = out_nbr + r * K;
    int* rd = out_dist + r * K;
    // reachable count and max distance
    int nreach = 0, maxd = 0;
    for (int u0 = 0; u0 < n; u0 += 32) {
      int u = u0 + lane;
      bool ok = u < n && u != v && R[u] != GU_INF32;
      if (ok) maxd = max(maxd, R[u]);
      nreach += __popc(__ballot_sync(FULL, ok));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) maxd = max(maxd, __shfl_xor_sync(FULL, maxd, o));
    int cnt = 0;
    if (nreach <= K) {
      for (int u0 = 0; u0 < n; u0 += 32) {
        int u = u0 + lane;
        bool ok = u < n && u != v && R[u] != GU_INF32;
        unsigned bal = __ballot_sync(FULL, ok);
        if (ok) {
          int q = cnt + __popc(bal & lanemask_lt());
          rn[q] = u;
          rd[q] = R[u];
        }
        cnt += __popc(bal);
      }
    } else {
      // kth = smallest d with #{reachable, R <= d} >= K (binary search on d)
      int lo = 0, hi = maxd;
      while (lo < hi) {
        int mid = lo + (hi - lo) / 2;
        int c = 0;
        for (int u0 = 0; u0 < n; u0 += 32) {
          int u = u0 + lane;
          bool ok = u < n && u != v && R[u] != GU_INF32 && R[u] <= mid;
          c += __popc(__ballot_sync(FULL, ok));
        }
        if (c >= K) hi = mid; else lo = mid + 1;
      }
      const int kth = lo;
      int T = 0;
      for (int u0 = 0; u0 < n; u0 += 32) {
        int u = u0 + lane;
        bool ok = u < n && u != v && R[u] != GU_INF32;
        bool lower = ok && R[u] < kth;
        bool tie = ok && R[u] == kth;
        unsigned bl = __ballot_sync(FULL, lower), bt = __ballot_sync(FULL, tie);
        if (lower) {
          int q = cnt + __popc(bl & lanemask_lt());
          rn[q] = u;
          rd[q] = R[u];
        }
        if (tie) ids[T + __popc(bt & lanemask_lt())] = u;
        cnt += __popc(bl);
        T += __popc(bt);
      }
      const int need = K - cnt;
      for (int i = lane; i < T; i += 32) perm[i] = i;
      __syncwarp();
      if (lane == 0) {
        Pcg64 rng;
        pcg64_from_seedseq(rng, seed, (unsigned long long)v);
        for (int i = T - 1; i >= 1; i--) {
          int j = (int)rng.interval((unsigned long long)i);
          int t = perm[i];
          perm[i] = perm[j];
          perm[j] = t;
        }
      }
      __syncwarp();
      for (int q = lane; q < need; q += 32) {
        rn[cnt + q] = ids[perm[q]];
        rd[cnt + q] = kth;
      }
      __syncwarp();
      cnt = K;
    }
    __syncwarp();
    // final (dist, id) order (lexsort((chosen, d)), neighbors.py:219)
    if (lane == 0) {
      for (int i = 1; i < cnt; i++) {
        int a = rn[i], d = rd[i], j = i - 1;
        while (j >= 0 && (rd[j] > d || (rd[j] == d && rn[j] > a))) {
          rn[j + 1] = rn[j];
          rd[j + 1] = rd[j];
          j--;
        }
        rn[j + 1] = a;
        rd[j + 1] = d;
      }
      out_cnt[r] = cnt;
    }
    __syncwarp();
  }
}

size_t slot_bytes_for(long long n, int L, bool knn) {
  size_t b = sizeof(unsigned long long) * (size_t)n * (size_t)(1 + L);
  if (knn) b += sizeof(int) * (size_t)n * FB_WARPS;
  return (b + 255) & ~(size_t)255;
}

int levels_for(int k, bool knn) { return knn ? k + 2 : 2; }

}  // namespace

// one stress pass over every source (metrics.cu); acc: >= ctas double2
int stress_bfs_pass(int64_t n, const int32_t* indptr, const int32_t* indices, const double* xy,
                    int pass2, const double* scale, void* acc, int* flag, void* workspace,
                    size_t ws_bytes, int ctas, const int32_t* sources, int64_t nsources,
                    cudaStream_t st) {
  const long long nsrc = sources ? nsources : n;
  const long long nbatches = (nsrc + 63) / 64;
  if (ctas > nbatches) ctas = (int)nbatches;
  if (ctas < 1) ctas = 1;
  const size_t slot = slot_bytes_for(n, levels_for(0, false), false);
  if (!workspace || ws_bytes < slot * (size_t)ctas) {
    set_error("stress BFS: workspace %zu < %zu", ws_bytes, slot * (size_t)ctas);
    return GU_ERR_WORKSPACE;
  }
  StressArgs sa{(const double2*)xy, scale, (double2*)acc, flag, pass2, sources};
  msbfs_kernel<MODE_STRESS><<<(unsigned)ctas, FB_THREADS, 0, st>>>(
      (int)n, indptr, indices, 0, 0, 0, nsrc, nullptr, nullptr, nullptr, nullptr,
      (char*)workspace, slot, levels_for(0, false), nullptr, sa);
  GU_CHECK_LAUNCH("msbfs_kernel<stress>");
  return GU_OK;
}

size_t stress_bfs_workspace(int64_t n, int ctas) {
  return slot_bytes_for(n, levels_for(0, false), false) * (size_t)(ctas > 0 ? ctas : 1);
}

}  // namespace gu

using namespace gu;

extern "C" size_t gu_full_bfs_workspace_size(int64_t n, int32_t k, int32_t batches_in_flight) {
  if (batches_in_flight < 1) batches_in_flight = 1;
  size_t a = slot_bytes_for(n, levels_for(k, true), true);
  size_t b = slot_bytes_for(n, levels_for(k, false), false);
  return (a > b ? a : b) * (size_t)batches_in_flight;
}

static int launch_msbfs(bool knn, int64_t n, const int32_t* indptr, const int32_t* indices,
                        int32_t k, uint64_t seed, int64_t src_begin, int64_t src_end,
                        int32_t* out_nbr, int32_t* out_dist, int32_t* out_count,
                        int32_t* out_rows, uint64_t* work, void* workspace, size_t ws_bytes,
                        int32_t bif, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 0 || n >= INT_MAX || src_begin < 0 || src_end > n || src_end < src_begin ||
      (knn && k < 0)) {
    set_error("full BFS: bad arguments");
    return GU_ERR_ARG;
  }
  if (bif < 1) bif = 1;
  const long long nsrc = src_end - src_begin;
  const long long nbatches = (nsrc + 63) / 64;
  if (bif > nbatches) bif = (int32_t)(nbatches > 0 ? nbatches : 1);
  const int L = levels_for(k, knn);
  const size_t slot = slot_bytes_for(n, L, knn);
  if (!workspace || ws_bytes < slot * (size_t)bif) {
    set_error("full BFS: workspace %zu < %zu", ws_bytes, slot * (size_t)bif);
    return GU_ERR_WORKSPACE;
  }
  if (work) GU_CHECK(cudaMemsetAsync(work, 0, 2 * sizeof(uint64_t), st));
  if (nsrc == 0) return GU_OK;
  if (knn && k == 0) {
    GU_CHECK(cudaMemsetAsync(out_count, 0, sizeof(int32_t) * nsrc, st));
    return GU_OK;
  }
  if (knn) {
    msbfs_kernel<MODE_KNN><<<(unsigned)bif, FB_THREADS, 0, st>>>(
        (int)n, indptr, indices, k, seed, src_begin, src_end, out_nbr, out_dist, out_count,
        nullptr, (char*)workspace, slot, L, (unsigned long long*)work, StressArgs{});
  } else {
    msbfs_kernel<MODE_APSP><<<(unsigned)bif, FB_THREADS, 0, st>>>(
        (int)n, indptr, indices, 0, 0, src_begin, src_end, nullptr, nullptr, nullptr, out_rows,
        (char*)workspace, slot, L, (unsigned long long*)work, StressArgs{});
  }
  GU_CHECK_LAUNCH("msbfs_kernel");
  return GU_OK;
}

extern "C" int gu_apsp_rows(int64_t n, const int32_t* indptr, const int32_t* indices,
                            int64_t src_begin, int64_t src_end, int32_t* out_rows,
                            void* workspace, size_t ws_bytes, int32_t batches_in_flight,
                            void* stream) {
  return launch_msbfs(false, n, indptr, indices, 0, 0, src_begin, src_end, nullptr, nullptr,
                      nullptr, out_rows, nullptr, workspace, ws_bytes, batches_in_flight, stream);
}

extern "C" int gu_full_bfs_knn(int64_t n, const int32_t* indptr, const int32_t* indices,
                               int32_t k, uint64_t seed, int64_t src_begin, int64_t src_end,
                               int32_t* out_nbr, int32_t* out_dist, int32_t* out_count,
                               uint64_t* work_counters, void* workspace, size_t ws_bytes,
                               int32_t batches_in_flight, void* stream) {
  return launch_msbfs(true, n, indptr, indices, k, seed, src_begin, src_end, out_nbr, out_dist,
                      out_count, nullptr, work_counters, workspace, ws_bytes, batches_in_flight,
                      stream);
}

extern "C" size_t gu_knn_from_rows_workspace_size(int64_t n, int32_t slots) {
  return sizeof(int32_t) * 2 * (size_t)n * (size_t)(slots > 0 ? slots : 1);
}

extern "C" int gu_knn_from_rows(int64_t n, const int32_t* rows, int64_t row_begin, int64_t nrows,
                                int32_t k, uint64_t seed, int32_t* out_nbr, int32_t* out_dist,
                                int32_t* out_count, void* workspace, size_t ws_bytes,
                                int32_t slots, void* stream) {
  if (slots < 1) slots = 1;
  if (n < 0 || n >= INT_MAX || k < 0 || nrows < 0) {
    set_error("gu_knn_from_rows: bad arguments");
    return GU_ERR_ARG;
  }
  if (ws_bytes < gu_knn_from_rows_workspace_size(n, slots)) {
    set_error("gu_knn_from_rows: workspace too small");
    return GU_ERR_WORKSPACE;
  }
  if (nrows == 0) return GU_OK;
  unsigned blocks = (unsigned)((slots * 32 + 255) / 256);
  knn_rows_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(
      (int)n, rows, row_begin, nrows, k, seed, out_nbr, out_dist, out_count, (int*)workspace,
      slots);
  GU_CHECK_LAUNCH("knn_rows_kernel");
  return GU_OK;
}
