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
// level L+1 in discovery order == the frontier's adjacency lists concatenated
// in queue order, each vertex kept at its first occurrence (equivalently: its
// vertices sorted by (min rank of a parent in level L, vertex id), SURVEY.md
// 8(a) A5).  Each warp expands a whole level at once (flattened adjacency of
// the frontier, 32 entries per step) against a shared-memory hash of the
// vertices already discovered, compacting first occurrences in order.
//
// Tiers (no host sync between them; overflow lists live in device memory):
//   tier F   register fast path: levels 1-2 reach k, deg(s) <= 32 (default)
//   tier 1a  lean warp per source, shared hash, CAP=128 discovered vertices
//   tier C   one 256-thread CTA per source, 4096-slot shared hash, CAP=3072
//            (hub-adjacent balls; ids < 2^23 - 1)
//   tier 1b  lean warp per source, shared hash, CAP=1024 (tier C's role
//            when ids >= 2^23 - 1)
//   tier 2   per-warp global stamp array of n ints, parents expanded
//            sequentially in queue order (any level size, any k)
// First occurrences within a chunk are found by packed (tag << 24 | id)
// keys and a shared atomicMin when ids < 2^24 - 1, by a MATCH election
// otherwise (a MATCH costs an ADU slot per distinct value: see tier F).
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "gumap.h"

namespace gu {
namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ unsigned hash_id(int w) { return (unsigned)w * 0x9E3779B1u; }
#ifndef PB_HASH_HIGH
#define PB_HASH_HIGH 1
#endif
// home slot of id w in a table of HC (a power of two) slots: the top bits of
// the Fibonacci product (PB_HASH_HIGH) or its low bits
template <int HC>
__device__ __forceinline__ unsigned hash_slot(int w) {
  constexpr int B = __builtin_ctz(HC);
  return PB_HASH_HIGH ? (hash_id(w) >> (32 - B)) : (hash_id(w) & (HC - 1));
}

// Tier-1 geometry: G lanes per source (32 / G sources per warp), at most CAP
// vertices discovered (hash of 2*CAP slots), PCAP frontier parents and TCAP
// flattened frontier adjacency entries per level.
template <int G, int CAP, int PCAP, int TCAP>
struct Tier1 {
  static constexpr int HC = 2 * CAP;
  static constexpr int TW = TCAP / 32;
  // per-group shared layout (ints): hkey[HC] disc[CAP] ppre[PCAP] pbeg[PCAP] bmap[TW]
  static constexpr int WORDS = HC + CAP + 2 * PCAP + TW;
  static constexpr int NG = 32 / G;
  static_assert(HC % 4 == 0 && (WORDS % 4) == 0, "int4 alignment");
};

// (i+1)-th output of the splitmix64 stream whose state starts at `base`
// (_kernels.py:18-25): draws are independent of each other, so the lanes of a
// group compute the crossing level's Fisher-Yates indices in parallel.
__device__ __forceinline__ unsigned long long splitmix_at(unsigned long long base, int i) {
  unsigned long long z = base + SPLIT_GAMMA * (unsigned long long)(i + 1);
  z = (z ^ (z >> 30)) * SPLIT_MUL1;
  z = (z ^ (z >> 27)) * SPLIT_MUL2;
  return z ^ (z >> 31);
}

// x % d for d < 2^31 without the 64-bit division routine: a double-precision
// quotient estimate (never above the true quotient, error < 2^14) corrected
// in exact integer arithmetic.
__device__ __forceinline__ int umod64_small(unsigned long long x, int d) {
  const double dd = (double)d;
  const unsigned long long q = (unsigned long long)__ddiv_rz(__ull2double_rz(x), dd);
  long long r = (long long)(x - q * (unsigned long long)d);  // 0 <= r < 2^14 * d
  const long long q2 = (long long)((double)r / dd);
  r -= q2 * (long long)d;
  while (r < 0) r += d;
  while (r >= d) r -= d;
  return (int)r;
}

// Discovery order without sorting: the reference appends a vertex the first
// time it is met while scanning the frontier in queue order, each parent's
// sorted adjacency in turn.  Concatenating the frontier's adjacency lists in
// that order (the "flattened" index t) and keeping each vertex at its first
// occurrence t -- and only if no earlier level holds it -- therefore yields
// the next level in exactly the reference's order.  The warp tiers
// below walk t in chunks of 32: the parent of t comes from adjacency-start
// bits (popc), __match_any_sync elects the lowest lane of equal ids inside a
// chunk, and that lane's atomicCAS into the per-source hash succeeds iff the
// id was never seen in an earlier chunk or level; ballot/popc compacts the
// winners in t order.

// Lean warp per source: tiers 1a (CAP 128) and 1b (CAP 1024), the fallbacks of
// the register fast path F for any ball shape and k <= 32.
//   * level 1 is the sorted adjacency of s itself: no dedupe beyond the hash
//     insert, and (when not crossing) already in output order;
//   * deeper levels: parent of a flattened index from a per-level bitmap of
//     adjacency starts (popc), the next chunk's candidate load issued before
//     the current chunk's hash work;
//   * a level's entries are written to the output row as soon as the level is
//     settled (rank by id inside the level; levels are in distance order);
//   * overflow is detected before the hash can fill, so probing is unbounded.
template <int CAP, int PCAP, int TCAP, int WARPS, int MINB, bool PACKED>
__global__ void __launch_bounds__(WARPS * 32, MINB)
    pbfs_warp(const int* __restrict__ indptr, const int* __restrict__ indices, int K,
              unsigned long long seed, long long src_begin, long long nsrc,
              const int* __restrict__ list, const int* __restrict__ list_count,
              int* __restrict__ out_nbr, int* __restrict__ out_dist, int* __restrict__ out_cnt,
              int* __restrict__ ovf_list, int* __restrict__ ovf_count,
              unsigned long long* __restrict__ work) {
  using L = Tier1<32, CAP, PCAP, TCAP>;
  constexpr int HC = L::HC, TW = L::TW;
  extern __shared__ __align__(16) int smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u, le_mask = (2u << lane) - 1u;
  int* const hkey = smem + warp * L::WORDS;
  int* const disc = hkey + HC;
  int* const ppre = disc + CAP;
  int* const pbeg = ppre + PCAP;
  unsigned* const bmap = reinterpret_cast<unsigned*>(pbeg + PCAP);
  unsigned long long w_scanned = 0, w_expanded = 0;

  // claim w in the hash; true iff it was not there (table never fills: the
  // callers stop inserting once a source is known to overflow CAP)
  auto claim = [&](int w) -> bool {
    unsigned h = hash_slot<HC>(w);
    for (;;) {
      const int old = atomicCAS(&hkey[h], -1, w);
      if (old == -1) return true;
      if (old == w) return false;
      h = (h + 1) & (HC - 1);
    }
  };

  const long long total = list ? (long long)(*list_count) : nsrc;
  for (long long it = (long long)blockIdx.x * WARPS + warp; it < total;
       it += (long long)gridDim.x * WARPS) {
    const int s = list ? list[it] : (int)(src_begin + it);
    const long long item = (long long)s - src_begin;  // output row
    int* const rn = out_nbr + item * K;
    int* const rd = out_dist + item * K;
    {
      int4* h4 = reinterpret_cast<int4*>(hkey);
#pragma unroll
      for (int i = lane; i < HC / 4; i += 32) h4[i] = make_int4(-1, -1, -1, -1);
    }
    const int b0 = __ldg(indptr + s);
    const int T0 = __ldg(indptr + s + 1) - b0;
    __syncwarp();
    const unsigned long long fy_base = seed + SPLIT_GAMMA * (unsigned long long)(s + 1);
    bool ovf = T0 > CAP - 2;
    int count = 0, nst = 0, lb = 1, le = 1, depth = 1;
    unsigned long long scanned = T0, expanded = 1;
    if (!ovf) {
      // ---- level 1: adjacency of s, already in discovery (= id) order
      if (lane == 0) hkey[hash_slot<HC>(s)] = s;
      __syncwarp();
      for (int t0 = 0; t0 < T0; t0 += 32) {
        const int t = t0 + lane;
        if (t < T0) {
          const int w = __ldg(indices + b0 + t);
          claim(w);
          disc[1 + t] = w;
        }
      }
      __syncwarp();
      nst = T0;
      le = 1 + T0;
      if (nst > K) {
        // level 1 crosses the budget: partial Fisher-Yates, picks ranked by id
        int j = 0;
        if (lane < K) j = lane + umod64_small(splitmix_at(fy_base, lane), nst - lane);
        for (int i = 0; i < K; i++) {
          const int ji = __shfl_sync(FULL, j, i);
          if (lane == 0) {
            const int a = disc[1 + i];
            disc[1 + i] = disc[1 + ji];
            disc[1 + ji] = a;
          }
        }
        __syncwarp();
        if (lane < K) {
          const int v = disc[1 + lane];
          int r = 0;
          for (int q = 0; q < K; q++) r += disc[1 + q] < v;
          rn[r] = v;
          rd[r] = 1;
        }
        count = K;
      } else {
        if (lane < nst) {
          rn[lane] = disc[1 + lane];
          rd[lane] = 1;
        }
        count = nst;
      }
    }
    // ---- deeper levels
    while (!ovf && count < K && nst > 0) {
      const int f = nst;  // frontier = last level, disc[lb, le)
      if (f > PCAP) {
        ovf = true;
        break;
      }
      for (int w = lane; w < TW; w += 32) bmap[w] = 0u;
      __syncwarp();
      int carry = 0, nne = 0;
      for (int i0 = 0; i0 < f; i0 += 32) {
        const int i = i0 + lane;
        int d = 0, b = 0;
        if (i < f) {
          const int u = disc[lb + i];
          b = __ldg(indptr + u);
          d = __ldg(indptr + u + 1) - b;
        }
        const int inc = warp_incl_scan(d);
        const unsigned ne = __ballot_sync(FULL, d > 0);
        if (d > 0) {
          const int r = nne + __popc(ne & lt);
          const int p0 = carry + inc - d;
          ppre[r] = p0;
          pbeg[r] = b;
          if (p0 < TCAP) atomicOr(&bmap[p0 >> 5], 1u << (p0 & 31));
        }
        carry += __shfl_sync(FULL, inc, 31);
        nne += __popc(ne);
      }
      const int T = carry;
      if (T > TCAP) {
        ovf = true;
        break;
      }
      __syncwarp();
      scanned += T;
      expanded += f;
      depth++;
      const int room = CAP - le;
      nst = 0;
      int pb = -1;
      unsigned m = T > 0 ? bmap[0] : 0u;
      int w = -1;
      if (lane < T) {
        const int p = pb + __popc(m & le_mask);
        w = __ldg(indices + pbeg[p] + (lane - ppre[p]));
      }
      pb += __popc(m);
      for (int t0 = 0; t0 < T; t0 += 32) {
        if (nst >= room) {  // the level cannot fit: stop inserting, overflow
          ovf = true;
          break;
        }
        int wn = -1;
        const int t1 = t0 + 32;
        if (t1 < T) {
          const unsigned m1 = bmap[t1 >> 5];
          if (t1 + lane < T) {
            const int p = pb + __popc(m1 & le_mask);
            wn = __ldg(indices + pbeg[p] + (t1 + lane - ppre[p]));
          }
          pb += __popc(m1);
        }
        bool isnew;
        if (PACKED) {
          // ids below 2^24 - 1: the chunk inserts (lane + 1) << 24 | id, equal
          // ids keep the lowest lane (atomicMin), settled ids hold tag 0; the
          // chunk's first occurrences then retag their slot to 0.  No MATCH
          // (one ADU slot per distinct id, see tier F).
          const bool valid = t0 + lane < T;
          const unsigned key = ((unsigned)(lane + 1) << 24) | (unsigned)w;
          unsigned h = hash_slot<HC>(w);
          unsigned old = valid ? (unsigned)atomicCAS(&hkey[h], -1, (int)key) : 0u;
          bool coll = valid && old != 0xffffffffu && (old & 0xffffffu) != (unsigned)w;
          if (__any_sync(FULL, coll)) {
            while (coll) {
              h = (h + 1) & (HC - 1);
              old = (unsigned)atomicCAS(&hkey[h], -1, (int)key);
              coll = old != 0xffffffffu && (old & 0xffffffu) != (unsigned)w;
            }
          }
          const bool mine = valid && (old == 0xffffffffu || (old >> 24) != 0u);
          if (mine && old != 0xffffffffu) atomicMin(reinterpret_cast<unsigned*>(&hkey[h]), key);
          __syncwarp();
          isnew = mine && (unsigned)hkey[h] == key;
          __syncwarp();
          if (isnew) hkey[h] = w;
        } else {
          const unsigned grp = __match_any_sync(FULL, w);
          isnew = t0 + lane < T && lane == __ffs(grp) - 1 && claim(w);
        }
        const unsigned bal = __ballot_sync(FULL, isnew);
        if (isnew) {
          const int pos = nst + __popc(bal & lt);
          if (pos < room) disc[le + pos] = w;
        }
        nst += __popc(bal);
        w = wn;
      }
      if (ovf || nst > room - 1) {
        ovf = true;
        break;
      }
      __syncwarp();
      if (nst == 0) break;
      const int remaining = K - count;
      int take = nst;
      if (nst > remaining) {
        int j = 0;
        if (lane < remaining) j = lane + umod64_small(splitmix_at(fy_base, lane), nst - lane);
        for (int i = 0; i < remaining; i++) {
          const int ji = __shfl_sync(FULL, j, i);
          if (lane == 0) {
            const int a = disc[le + i];
            disc[le + i] = disc[le + ji];
            disc[le + ji] = a;
          }
        }
        __syncwarp();
        take = remaining;
      }
      for (int i0 = 0; i0 < take; i0 += 32) {
        const int i = i0 + lane;
        if (i < take) {
          const int v = disc[le + i];
          int r = 0;
          for (int q = 0; q < take; q++) r += disc[le + q] < v;
          rn[count + r] = v;
          rd[count + r] = depth;
        }
      }
      count += take;
      lb = le;
      le += nst;
    }
    if (ovf) {
      if (lane == 0) ovf_list[atomicAdd(ovf_count, 1)] = s;
      continue;
    }
    if (lane == 0) out_cnt[item] = count;
    w_scanned += scanned;
    w_expanded += expanded;
  }
  if (work && lane == 0) {
    atomicAdd(work, w_scanned);
    atomicAdd(work + 1, w_expanded);
  }
}

// ---------------------------------------------------------- tier F (fast)
// The dominant shape of a k-ball on the BASELINE graphs: level 1 (the sorted
// adjacency of s, <= 32 ids) and level 2 crossing the budget.  Everything is
// kept in registers: lane i holds parent i of level 2 (= the i-th neighbour of
// s); zero-degree parents are compacted away by ballot; the parent of a
// flattened index t is the number of adjacency starts <= t inside the chunk
// (__reduce_or_sync of per-parent bits) plus the starts of earlier chunks,
// fetched by shuffle; the next chunk's loads are issued before the current
// chunk's hash work.  Sources of any other shape (deg(s) > 32, a level 2 that
// does not reach k, a ball above the budget) go to the generic tiers.
#ifndef TF_CAP2
#define TF_CAP2 160  // level-2 ids kept per source
#endif
#ifndef TF_HC
#define TF_HC 512  // hash slots per source (ball budget 3/4 of it)
#endif

// M_d = ceil(2^64 / d), 2 <= d <= 4096, for the table remainder: a constant
// initialiser in the image (no upload, no host-side state)
struct MagicTab {
  unsigned long long v[4097];
  constexpr MagicTab() : v() {
    for (int d = 2; d <= 4096; d++) v[d] = ~0ull / (unsigned long long)d + 1ull;
  }
};
__device__ const MagicTab g_magic = MagicTab();

// 64-bit remainder by a small divisor (1 <= d <= 4096): q = mulhi(x, M_d) with
// M_d = ceil(2^64 / d) is floor(x / d) or one more (Granlund-Montgomery), so a
// single conditional correction gives the exact x % d.
__device__ __forceinline__ int umod64_tab(unsigned long long x, int d) {
  if (d == 1) return 0;
  const unsigned long long q = __umul64hi(x, __ldg(&g_magic.v[d]));
  unsigned long long r = x - q * (unsigned long long)d;
  if (r > x) r += (unsigned long long)d;  // q was one too large
  return (int)r;
}

#ifndef TF_MINB
#define TF_MINB 8
#endif
#ifndef TF_NO_INNER_SYNC
#define TF_NO_INNER_SYNC 1  // the warp barrier before the read-back orders the atomics; none needed after the probe loops
#endif
#ifndef TF_PRED_STORE
#define TF_PRED_STORE 1  // predicated list stores (no sink-word wavefronts for lanes with nothing new)
#endif
#ifndef TF_MERGED_VOTE
#define TF_MERGED_VOTE 1  // one probe-loop vote per chunk pair
#endif
constexpr int TH_DMIN = 64;  // tier H: smallest degree of an implicit (hub) parent

// Partial Fisher-Yates in closed form.  Lane i < r holds its draw j_i (>= i)
// of the reference's sequential swaps swap(a[i], a[j_i]), i = 0..r-1
// (_kernels.py:98-105); returns the ORIGINAL position whose value ends in
// slot i.  Slot i is never touched after step i, so it receives what position
// j_i held just before step i: the value the last earlier step with the same
// draw moved there (lanes of equal draws: one MATCH; inactive lanes share
// one key, so it costs at most r + 1 ADU slots), else a[j_i] itself.  What a
// position k < r held just before step k is, likewise, what the last earlier
// step drawing k moved there: a chain k -> W(k) -> ... ending at an original
// position, resolved by pointer jumping (draws rarely collide).  wsc: 32
// ints of per-warp scratch.
__device__ __forceinline__ int fy_positions(int r, int lane, int j, int* wsc) {
  const bool act = lane < r;
  const unsigned grp = __match_any_sync(FULL, act ? j : -1);
  wsc[lane] = lane;
  __syncwarp();
  // W(d) = the last step i < d with j_i == d: the member of d's draw group
  // with no other member strictly between it and d
  if (act && j < r && j > lane && (grp & ~((2u << lane) - 1u) & ((1u << j) - 1u)) == 0) wsc[j] = lane;
  __syncwarp();
  int nxt = wsc[lane];
  for (;;) {
    const int n2 = __shfl_sync(FULL, nxt, nxt);
    if (!__any_sync(FULL, n2 != nxt)) break;
    nxt = n2;
  }
  const unsigned prev = act ? grp & ((1u << lane) - 1u) : 0u;
  const int vL = __shfl_sync(FULL, nxt, (31 - __clz(prev)) & 31);
  return prev ? vL : j;
}

// inclusive warp scan: the validity predicate of shfl.up replaces the
// per-step lane test
template <int O>
__device__ __forceinline__ void scan_step(int& v) {
  asm("{\n\t.reg .s32 t;\n\t.reg .pred p;\n\t"
      "shfl.sync.up.b32 t|p, %0, %1, 0, -1;\n\t"
      "@p add.s32 %0, %0, t;\n\t}"
      : "+r"(v)
      : "n"(O));
}
__device__ __forceinline__ int warp_incl_scan_p(int v) {
  scan_step<1>(v);
  scan_step<2>(v);
  scan_step<4>(v);
  scan_step<8>(v);
  scan_step<16>(v);
  return v;
}

// rank of v among the (distinct) values of lanes 0..r-1
__device__ __forceinline__ int rank_in_warp(int r, int v) {
  if (r <= 8) {
    // all r * r comparisons at once: lane L compares value L >> 2 with the
    // values of lanes L & 3 and (L & 3) + 4; lane i < r sums the bits of
    // lanes 4i .. 4i + 3 of both ballots (one step instead of r shuffles)
    const int lane = threadIdx.x & 31;
    const int q = lane & 3;
    const int vi = __shfl_sync(FULL, v, lane >> 2);
    const int va = __shfl_sync(FULL, v, q);
    const int vb = __shfl_sync(FULL, v, q + 4);
    const unsigned ba = __ballot_sync(FULL, q < r && va < vi);
    const unsigned bb = __ballot_sync(FULL, q + 4 < r && vb < vi);
    const unsigned m = 0xfu << ((lane & 7) << 2);
    return __popc(ba & m) + __popc(bb & m);
  }
  int rk = 0;
  for (int q = 0; q < r; q++) rk += __shfl_sync(FULL, v, q) < v;
  return rk;
}

// PACKED (n < 2^24 - 1): hash slots hold (tag << 24 | id) and duplicates
// inside a chunk pair are resolved by a shared-memory atomicMin on the tag
// (the flattened position t + 1): no MATCH.  A MATCH.ANY occupies the ADU one
// slot per DISTINCT value among the lanes (~64 SM cycles for 32 distinct ids,
// profiles/r02_micro_adu.log), and the ADU was the most-used pipe of this
// kernel (73%).  !PACKED keeps the MATCH election for larger graphs.
template <int WARPS, bool PACKED>
__global__ void __launch_bounds__(WARPS * 32, TF_MINB)
    pbfs_fast(const int* __restrict__ indptr, const int* __restrict__ indices, int K,
              unsigned long long seed, long long src_begin, long long nsrc,
              int* __restrict__ out_nbr, int* __restrict__ out_dist, int* __restrict__ out_cnt,
              int* __restrict__ ovf_list, int* __restrict__ ovf_count,
              int* __restrict__ hub_list, int* __restrict__ hub_count, int* __restrict__ hub_direct,
              unsigned long long* __restrict__ work) {
  constexpr int HC = TF_HC;
  __shared__ __align__(16) int sm_hash[WARPS][HC];
  // +32: a chunk never writes past; +32 more: per-lane sink for the
  // unconditional (branch-free) list store of lanes with nothing new
  __shared__ int sm_list[WARPS][TF_CAP2 + 64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u, le_mask = (2u << lane) - 1u;
  int* const hkey = sm_hash[warp];
  int* const lst = sm_list[warp];
  const unsigned hbase = (unsigned)__cvta_generic_to_shared(hkey);
  // per-warp work counters: < 2^31 sources / 2^16 warps * 286 entries fits 32 bits
  unsigned w_scanned = 0, w_expanded = 0;
  static_assert(TF_CAP2 + 32 + 1 + 32 <= (HC * 3) / 4, "ball budget must fit the hash");
  // Warp-wide claim of distinct keys (one per lane, `lead` lanes only): one
  // predicated CAS for everybody; the linear-probe loop runs only when some
  // lane hit an occupied slot, so the common case has no divergence.
  auto claim = [&](int w, bool lead) -> bool {
    unsigned h = hash_slot<HC>(w);
    int old = w;  // predicated CAS (no branch): lanes with !lead keep old == w
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\t"
        "@p atom.shared.cas.b32 %0, [%2], -1, %3;\n\t}"
        : "+r"(old)
        : "r"((unsigned)lead), "r"(hbase + 4u * h), "r"(w)
        : "memory");
    bool coll = old != -1 && old != w;
    if (__any_sync(FULL, coll)) {
      while (coll) {
        h = (h + 1) & (HC - 1);
        old = atomicCAS(&hkey[h], -1, w);
        coll = old != -1 && old != w;
      }
      __syncwarp();
    }
    return lead && old == -1;
  };
  // 32-bit source index: nsrc < 2^31 and the grid stride is below 2^20
  for (unsigned item = blockIdx.x * WARPS + warp; item < (unsigned)nsrc;
       item += gridDim.x * WARPS) {
    const int s = (int)src_begin + (int)item;
    int* const rn = out_nbr + (size_t)item * K;
    int* const rd = out_dist + (size_t)item * K;
    const int b0 = __ldg(indptr + s);
    const int T0 = __ldg(indptr + s + 1) - b0;
    if (T0 > 32) {
      if (lane == 0) ovf_list[atomicAdd(ovf_count, 1)] = s;
      continue;
    }
    const int w1 = lane < T0 ? __ldg(indices + b0 + lane) : -1;
    // level-2 parent ranges issued right away (needed unless level 1 crosses)
    int pb = 0, pd = 0;
    if (T0 < K && lane < T0) {
      pb = __ldg(indptr + w1);
      pd = __ldg(indptr + w1 + 1) - pb;
    }
    const unsigned long long fy_base = seed + SPLIT_GAMMA * (unsigned long long)(s + 1);
    if (T0 >= K) {
      // ---- level 1 reaches the budget: sorted adjacency, or a random subset
      // (no hash: nothing beyond level 1 is discovered)
      if (T0 == K) {
        if (lane < K) {
          rn[lane] = w1;
          rd[lane] = 1;
        }
      } else {
        // Fisher-Yates on positions of the sorted adjacency: the picks'
        // id order is their position order, so the rank is one popcount
        // (lane p holds position p: it stores its own id at rank
        // popc(picked positions below p))
        int j = lane;
        if (lane < K) j = lane + umod64_tab(splitmix_at(fy_base, lane), T0 - lane);
        const int P = fy_positions(K, lane, j, lst + TF_CAP2 + 32);
        const unsigned M = __reduce_or_sync(FULL, lane < K ? 1u << P : 0u);
        if ((M >> lane) & 1u) {
          const int r = __popc(M & lt);
          rn[r] = w1;
          rd[r] = 1;
        }
      }
      if (lane == 0) out_cnt[item] = T0 < K ? T0 : K;
      w_scanned += T0;
      w_expanded += 1;
      __syncwarp();
      continue;
    }
    if (T0 == 0) {  // isolated vertex: nothing reachable
      if (lane == 0) out_cnt[item] = 0;
      w_expanded += 1;
      continue;
    }
    // ---- level 1 in full
    if (lane < T0) {
      rn[lane] = w1;
      rd[lane] = 1;
    }
#pragma unroll
    for (int i = 0; i < HC / 128; i++) reinterpret_cast<int4*>(hkey)[lane + 32 * i] = make_int4(-1, -1, -1, -1);
    __syncwarp();
    // s itself rides on lane T0 (T0 < K <= 32) of the level-1 claim
    claim(lane == T0 ? s : w1, lane <= T0);
    // ---- level 2: prefix of the parents' degrees.  In an undirected CSR a
    // neighbour of s has s in its own list, so every parent is non-empty; a
    // CSR that breaks this (one-sided entries) takes the generic tiers.
    // One vote for both exits: an empty parent, or (PACKED) a level too
    // long for the 8-bit tags t + 1.
    const int nne = T0;
    const int cb = pb, cdv = pd;
    const int inc = warp_incl_scan_p(cdv);
    const int cpre = inc - cdv;
    const int T = __shfl_sync(FULL, inc, 31);
    if (__any_sync(FULL, (lane < T0 && pd <= 0) || (PACKED && T > 254))) {
      // a long level next to a high-degree parent: straight to the hub tier
      // (tier 1a would scan the hub's row only to overflow)
      const bool hub = hub_list && !__any_sync(FULL, lane < T0 && pd <= 0) &&
                       __reduce_max_sync(FULL, pd) >= TH_DMIN;
      if (lane == 0) {
        if (hub) {
          hub_list[atomicAdd(hub_count, 1)] = s;
          atomicAdd(hub_direct, 1);
        } else {
          ovf_list[atomicAdd(ovf_count, 1)] = s;
        }
      }
      continue;
    }
    int nst = 0, pcount = 0;
    // candidate of chunk t0 for this lane (parent count of earlier chunks: pc);
    // cbase = adjacency start - flattened start of the lane's parent, so a
    // candidate address is one shuffle and one add away
    const int cbase = cb - cpre;
    const int cpre_s = lane < nne ? cpre : 0x40000000;
    // Raw candidate ids of chunk t0 (parent count of earlier chunks: pc).
    // Lanes past T load indices[0] and keep it: they sit above every valid
    // lane, so they are never a first occurrence and never claim.
    auto load_chunk = [&](int t0, int pc, int& x, unsigned& m) {
      // PTX shl clamps shifts >= 32 to a zero result: parents outside the
      // chunk (off < 0 or >= 32, and the lanes past nne via cpre_s) add no bit
      unsigned bit;
      asm("shl.b32 %0, 1, %1;" : "=r"(bit) : "r"((unsigned)(cpre_s - t0)));
      m = __reduce_or_sync(FULL, bit);
      const int p = pc + __popc(m & le_mask) - 1;
      // 32-bit offset arithmetic (cbase may be negative; the sum never is)
      const unsigned base = (unsigned)__shfl_sync(FULL, cbase, p & 31);
      const int t = t0 + lane;
      x = __ldg(indices + (t < T ? base + (unsigned)t : 0u));
    };
    // claim the first occurrences (queue order) of chunks t0 and t0 + 32 (when
    // that one exists) and append them; true when the ball leaves the budget
    // (the hash holds it: static_assert).  Both MATCHes are issued before the
    // claims, and the second chunk's claims follow the first's, so each pair
    // costs one dependent round trip instead of two.
    // PACKED: insert one tagged key per lane (valid lanes only); h is the
    // slot holding the id, mine is true when the id was not in the hash
    // before this chunk pair (then the smallest tag of the pair wins the slot)
    auto insert_tagged = [&](int w, unsigned key, bool valid, unsigned base_tag, unsigned& h,
                             bool& mine) {
      // Predicated CAS (an unconditional one with a never-matching compare
      // value was 20% slower: lanes past T all hold the same id, so their
      // CASes serialise on one slot); the probe loop runs only when some lane
      // hit another id's slot.
      // Invalid lanes keep old = w (their own id with tag 0): neither a
      // collision nor a first occurrence, with no test of `valid` below; the
      // empty key's tag (255) is above every base tag.
      h = hash_slot<HC>(w);
      unsigned old = (unsigned)w;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\t"
          "@p atom.shared.cas.b32 %0, [%2], -1, %3;\n\t}"
          : "+r"(old)
          : "r"((unsigned)valid), "r"(hbase + 4u * h), "r"(key)
          : "memory");
      bool coll = old != 0xffffffffu && ((old ^ (unsigned)w) << 8) != 0u;
      if (__any_sync(FULL, coll)) {
        while (coll) {
          h = (h + 1) & (HC - 1);
          old = (unsigned)atomicCAS(&hkey[h], -1, (int)key);
          coll = old != 0xffffffffu && ((old ^ (unsigned)w) << 8) != 0u;
        }
        __syncwarp();
      }
      mine = (old >> 24) >= base_tag;
      // predicated RED (no branch, no wavefronts for the idle lanes): only
      // the lanes that met their id inserted earlier in this pair lower the
      // slot's tag (c5 with the pair-rank and shl changes: 2.76 -> 2.58 ms)
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, 0;\n\t"
          "@p red.shared.min.u32 [%1], %2;\n\t}"
          :
          : "r"((unsigned)(mine && old != 0xffffffffu)), "r"(hbase + 4u * h), "r"(key)
          : "memory");
    };
    auto process2p = [&](int t0, int xa, int xb) -> bool {
#if !TF_MERGED_VOTE
      const bool two = t0 + 32 < T;  // warp-uniform
#endif
      const unsigned base_tag = (unsigned)(t0 + 1);
      const unsigned ka = ((unsigned)(t0 + lane + 1) << 24) | (unsigned)xa;
      const unsigned kb = ((unsigned)(t0 + 33 + lane) << 24) | (unsigned)xb;
#if TF_MERGED_VOTE
      // both chunks' CASes first, ONE vote for their probe loops (insertion
      // order is free: equal ids settle on the smallest tag whatever the order)
      unsigned ha = hash_slot<HC>(xa), hb = hash_slot<HC>(xb);
      unsigned olda = (unsigned)xa, oldb = (unsigned)xb;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\t"
          "@p atom.shared.cas.b32 %0, [%2], -1, %3;\n\t}"
          : "+r"(olda)
          : "r"((unsigned)(t0 + lane < T)), "r"(hbase + 4u * ha), "r"(ka)
          : "memory");
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\t"
          "@p atom.shared.cas.b32 %0, [%2], -1, %3;\n\t}"
          : "+r"(oldb)
          : "r"((unsigned)(t0 + 32 + lane < T)), "r"(hbase + 4u * hb), "r"(kb)
          : "memory");
      bool ca = olda != 0xffffffffu && ((olda ^ (unsigned)xa) << 8) != 0u;
      bool cb = oldb != 0xffffffffu && ((oldb ^ (unsigned)xb) << 8) != 0u;
      if (__any_sync(FULL, ca || cb)) {
        while (ca) {
          ha = (ha + 1) & (HC - 1);
          olda = (unsigned)atomicCAS(&hkey[ha], -1, (int)ka);
          ca = olda != 0xffffffffu && ((olda ^ (unsigned)xa) << 8) != 0u;
        }
        while (cb) {
          hb = (hb + 1) & (HC - 1);
          oldb = (unsigned)atomicCAS(&hkey[hb], -1, (int)kb);
          cb = oldb != 0xffffffffu && ((oldb ^ (unsigned)xb) << 8) != 0u;
        }
#if !TF_NO_INNER_SYNC
        __syncwarp();
#endif
      }
      // (tag >= base tag, compared on whole keys: the tag is the top byte)
      const bool ma = olda >= (base_tag << 24), mb = oldb >= (base_tag << 24);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, 0;\n\t"
          "@p red.shared.min.u32 [%1], %2;\n\t}"
          :
          : "r"((unsigned)(ma && olda != 0xffffffffu)), "r"(hbase + 4u * ha), "r"(ka)
          : "memory");
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, 0;\n\t"
          "@p red.shared.min.u32 [%1], %2;\n\t}"
          :
          : "r"((unsigned)(mb && oldb != 0xffffffffu)), "r"(hbase + 4u * hb), "r"(kb)
          : "memory");
#else
      unsigned ha, hb;
      bool ma, mb;
      insert_tagged(xa, ka, t0 + lane < T, base_tag, ha, ma);
      insert_tagged(xb, kb, two && t0 + 32 + lane < T, base_tag, hb, mb);
#endif
      __syncwarp();
      const bool na = ma && (unsigned)hkey[ha] == ka;
      const bool nb = mb && (unsigned)hkey[hb] == kb;
      const unsigned ba = __ballot_sync(FULL, na);
      const unsigned bb = __ballot_sync(FULL, nb);
      // nst <= TF_CAP2 on entry: a's entries end below TF_CAP2 + 32, b's
      // below TF_CAP2 + 64 (past TF_CAP2 only when overflowing, which
      // discards the list); lanes with nothing new hit their sink
#if TF_PRED_STORE
      if (na) lst[nst + __popc(ba & lt)] = xa;
      nst += __popc(ba);
      if (nb) lst[nst + __popc(bb & lt)] = xb;
#else
      lst[na ? nst + __popc(ba & lt) : TF_CAP2 + 32 + lane] = xa;
      nst += __popc(ba);
      lst[nb ? nst + __popc(bb & lt) : TF_CAP2 + 32 + lane] = xb;
#endif
      nst += __popc(bb);
      return nst > TF_CAP2;
    };
    auto process2 = [&](int t0, int xa, int xb) -> bool {
      if (PACKED) return process2p(t0, xa, xb);
      const bool two = t0 + 32 < T;  // warp-uniform
      const unsigned ga = __match_any_sync(FULL, xa);
      const unsigned gb = two ? __match_any_sync(FULL, xb) : 0u;
      const bool na = claim(xa, t0 + lane < T && (ga & lt) == 0);
      const unsigned ba = __ballot_sync(FULL, na);
      // nst <= TF_CAP2 here: in bounds; lanes with nothing new hit their sink
      lst[na ? nst + __popc(ba & lt) : TF_CAP2 + 32 + lane] = xa;
      nst += __popc(ba);
      if (!two) return nst > TF_CAP2;
      if (nst > TF_CAP2) return true;
      __syncwarp();  // chunk a's claims are visible to chunk b's
      const bool nb = claim(xb, t0 + 32 + lane < T && (gb & lt) == 0);
      const unsigned bb = __ballot_sync(FULL, nb);
      lst[nb ? nst + __popc(bb & lt) : TF_CAP2 + 32 + lane] = xb;
      nst += __popc(bb);
      return nst > TF_CAP2;
    };
    // chunk registers in ping-pong pairs (unrolled by hand): the loads of the
    // next pair stay in flight while this pair is processed -- no register
    // move or select touches an in-flight load result
    int x0 = 0, x1 = 0, x2 = 0, x3 = 0;
    unsigned m0 = 0, m1 = 0, m2 = 0, m3 = 0;
    bool ovf = false;
    load_chunk(0, 0, x0, m0);
    pcount = __popc(m0);
    if (32 < T) {
      load_chunk(32, pcount, x1, m1);
      pcount += __popc(m1);
    }
    for (int t0 = 0;;) {
      if (t0 + 64 < T) {
        load_chunk(t0 + 64, pcount, x2, m2);
        pcount += __popc(m2);
        if (t0 + 96 < T) {
          load_chunk(t0 + 96, pcount, x3, m3);
          pcount += __popc(m3);
        }
      }
      if (process2(t0, x0, x1)) { ovf = true; break; }
      t0 += 64;
      if (t0 >= T) break;
      if (t0 + 64 < T) {
        load_chunk(t0 + 64, pcount, x0, m0);
        pcount += __popc(m0);
        if (t0 + 96 < T) {
          load_chunk(t0 + 96, pcount, x1, m1);
          pcount += __popc(m1);
        }
      }
      if (process2(t0, x2, x3)) { ovf = true; break; }
      t0 += 64;
      if (t0 >= T) break;
    }
    const int remaining = K - T0;
    if (ovf || nst < remaining) {  // level 2 does not reach k (or too big): generic path
      // a ball above this tier's budget is above tier 1a's too: hand it to
      // the hub tier (which passes what it cannot take on to the big-ball tiers)
      const bool hub = ovf && hub_list;
      if (lane == 0) {
        if (hub) {
          hub_list[atomicAdd(hub_count, 1)] = s;
          atomicAdd(hub_direct, 1);
        } else {
          ovf_list[atomicAdd(ovf_count, 1)] = s;
        }
      }
      __syncwarp();
      continue;
    }
    __syncwarp();
    int pos = lane;
    if (nst > remaining && lane < remaining)
      pos = lane + umod64_tab(splitmix_at(fy_base, lane), nst - lane);
    // one pick (remaining == 1): its draw is its position
    if (nst > remaining && remaining > 1) pos = fy_positions(remaining, lane, pos, lst + TF_CAP2 + 32);
    const int v = lst[pos];
    const int r = rank_in_warp(remaining, v);
    if (lane < remaining) {
      rn[T0 + r] = v;
      rd[T0 + r] = 2;
    }
    if (lane == 0) out_cnt[item] = K;
    w_scanned += (unsigned)(T0 + T);
    w_expanded += (unsigned)(1 + T0);
    __syncwarp();
  }
  if (work && lane == 0) {
    atomicAdd(work, (unsigned long long)w_scanned);
    atomicAdd(work + 1, (unsigned long long)w_expanded);
  }
}

// ------------------------------------------------------------- tier H (hub)
// Sources next to ONE high-degree vertex (scale-free graphs): level 2 is
// dominated by the hub's adjacency list N(H) (hundreds to thousands of ids),
// which tiers 1a / C scan and hash in full for every such source.  Here the
// hub's list is never scanned.  With H the largest-degree parent, level 2 in
// discovery order is
//   A    = first occurrences among the parents before H        (explicit)
//   hubs = N(H) \ X in id order, X = ({s} + N(s) + A) within N(H)  (implicit)
//   B    = first occurrences among the parents after H, outside N(H) (explicit)
// because N(H) is sorted and duplicate-free, and a vertex of N(H) is new
// unless an earlier part of the ball holds it.  Membership x in N(H) is tested
// as H in N(x) (the graph is undirected; N(x) is short), the members' ranks in
// N(H) by a 32-ary cooperative search; |hubs| = deg(H) - |X| >= 32 > k - T0,
// so level 2 is always the crossing level, n2 = |A| + |hubs| + |B|, and the
// Fisher-Yates picks (closed form, as tier F) index the three parts without
// materialising the middle one: position q of `hubs` is N(H)[q + #(X-ranks
// skipped)].  Work per source: O(explicit entries + |X| + k) instead of
// O(deg(H)).  Sources with other shapes (no big parent, a second hub that
// overflows the explicit list, > 32 members of X) go on to tier C / 1b.
#ifndef TH_HC
#define TH_HC 512
#endif
#ifndef TH_LCAP
#define TH_LCAP 160
#endif
constexpr int TH_WARPS = 8, TH_XCAP = 32;
#ifndef TH_MINB
#define TH_MINB 6
#endif
struct TierH {
  // hkey[HC] lst[LCAP + 32] cpre[32] cb[32] xs[32] wsc[32]
  static constexpr int WORDS = TH_HC + TH_LCAP + 32 + 4 * 32;
};
static_assert(1 + 31 + TH_LCAP + 32 <= (TH_HC * 3) / 4, "explicit ball must fit the hash");

// H in the sorted row indices[b, b + d)?  Long rows (another hub's) narrow
// 8-fold per round trip: seven independent pivot loads per step.
__device__ __forceinline__ bool row_has(const int* __restrict__ indices, int b, int d, int H) {
  int lo = b, len = d;
  while (len > 8) {
    const int step = (len + 7) >> 3;
    int c = 0;  // blocks [lo + i * step, +step) entirely below H form a prefix
#pragma unroll
    for (int i = 0; i < 7; i++) {
      const int last = lo + (i + 1) * step - 1;
      c += last < lo + len && __ldg(indices + last) < H;
    }
    lo += c * step;
    len = min(step, len - c * step);
  }
  bool f = false;
#pragma unroll
  for (int q = 0; q < 8; q++) f |= q < len && __ldg(indices + lo + q) == H;
  return f;
}

// ranks of up to 4 members x[0..m) in the sorted row nh[0, D): the warp
// narrows every member's range 32-fold per step, the loads of the members of
// a step in flight together (two round trips for D <= 1024)
__device__ __forceinline__ void hub_rank4(const int* __restrict__ nh, int D, const int (&x)[4], int m,
                                          int lane, int (&rank)[4]) {
  int lo[4], hi[4];
#pragma unroll
  for (int i = 0; i < 4; i++) {
    lo[i] = 0;
    hi[i] = i < m ? D : 0;
  }
  for (int span = D; span > 32;) {  // every live range has this length bound
    const int step = (span + 31) >> 5;
    int v[4];
#pragma unroll
    for (int i = 0; i < 4; i++) {
      const int bl = lo[i] + lane * step;
      v[i] = bl < hi[i] ? __ldg(nh + min(bl + step, hi[i]) - 1) : INT_MAX;
    }
#pragma unroll
    for (int i = 0; i < 4; i++) {
      const int c = __popc(__ballot_sync(FULL, v[i] < x[i]));  // blocks entirely below x
      lo[i] += c * step;
      hi[i] = min(lo[i] + step, hi[i]);
    }
    span = step;
  }
  int v[4];
#pragma unroll
  for (int i = 0; i < 4; i++) v[i] = lo[i] + lane < hi[i] ? __ldg(nh + lo[i] + lane) : INT_MAX;
#pragma unroll
  for (int i = 0; i < 4; i++) rank[i] = lo[i] + __popc(__ballot_sync(FULL, v[i] < x[i]));
}

__global__ void __launch_bounds__(TH_WARPS * 32, TH_MINB)
    pbfs_hub(const int* __restrict__ indptr, const int* __restrict__ indices, int K,
             unsigned long long seed, long long src_begin, const int* __restrict__ list,
             const int* __restrict__ list_count, int* __restrict__ out_nbr,
             int* __restrict__ out_dist, int* __restrict__ out_cnt, int* __restrict__ ovf_list,
             int* __restrict__ ovf_count, int* __restrict__ queue,
             unsigned long long* __restrict__ work) {
  constexpr int HC = TH_HC;
  extern __shared__ __align__(16) int smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  int* const hkey = smem + warp * TierH::WORDS;
  int* const lst = hkey + HC;
  int* const cpre_sh = lst + TH_LCAP + 32;
  int* const cb_sh = cpre_sh + 32;
  int* const xs = cb_sh + 32;
  int* const wsc = xs + 32;
  unsigned long long w_scanned = 0, w_expanded = 0;
  const int total = *list_count;
  if (total == 0) return;  // (no storm of queue atomics for an empty list)
  // sources are handed out one at a time (per-source latency varies a lot and
  // the list is only a few rounds of the resident warps long)
  for (;;) {
    int it = 0;
    if (lane == 0) it = atomicAdd(queue, 1);
    it = __shfl_sync(FULL, it, 0);
    if (it >= total) break;
    const int s = __ldg(list + it);
    const long long item = (long long)s - src_begin;
    int* const rn = out_nbr + item * K;
    int* const rd = out_dist + item * K;
    const int b0 = __ldg(indptr + s);
    const int T0 = __ldg(indptr + s + 1) - b0;
    bool ok = T0 >= 1 && T0 < K && T0 <= 31;
    int w1 = -1, pb = 0, pd = 0;
    if (ok && lane < T0) {
      w1 = __ldg(indices + b0 + lane);
      pb = __ldg(indptr + w1);
      pd = __ldg(indptr + w1 + 1) - pb;
    }
    // the hub: the largest-degree parent (lowest lane among equals)
    const int D = __reduce_max_sync(FULL, pd);
    const int hl = __ffs(__ballot_sync(FULL, lane < T0 && pd == D)) - 1;
    if (__any_sync(FULL, lane < T0 && pd <= 0) || D < TH_DMIN) ok = false;
    if (!ok) {
      if (lane == 0) ovf_list[atomicAdd(ovf_count, 1)] = s;
      continue;
    }
    const int H = __shfl_sync(FULL, w1, hl);
    const int* const nh = indices + __shfl_sync(FULL, pb, hl);
    // flattened adjacency of the explicit parents (the hub contributes nothing)
    const int pde = lane == hl ? 0 : pd;
    const int inc = warp_incl_scan(pde);
    const int Ts = __shfl_sync(FULL, inc, 31);
    const int Tsplit = __shfl_sync(FULL, inc - pde, hl);  // entries of the parents before H
    __syncwarp();  // the previous source's reads of the tables are done
    cpre_sh[lane] = lane < T0 ? inc - pde : INT_MAX;
    cb_sh[lane] = pb;
#pragma unroll
    for (int i = 0; i < HC / 128; i++)
      reinterpret_cast<int4*>(hkey)[lane + 32 * i] = make_int4(-1, -1, -1, -1);
    __syncwarp();
    if (lane <= T0) {  // s and level 1: distinct ids, tag 0
      const int w = lane == T0 ? s : w1;
      unsigned h = hash_slot<HC>(w);
      while (atomicCAS(&hkey[h], -1, w) != -1) h = (h + 1) & (HC - 1);
    }
    __syncwarp();
    int nl = 0;
    // first occurrences of flattened entries [tbeg, tend) appended to lst in
    // order (tier 1a's packed lane-tag claim); false: the list overflows
    auto expand = [&](int tbeg, int tend) -> bool {
      // candidate id of flattened entry t (parent by a search of the prefix table)
      auto cand = [&](int t) -> int {
        if (t >= tend) return 0;
        int p = 0;
#pragma unroll
        for (int st = 16; st; st >>= 1)
          if (cpre_sh[p + st] <= t) p += st;
        return __ldg(indices + cb_sh[p] + (t - cpre_sh[p]));
      };
      int wn = tbeg < tend ? cand(tbeg + lane) : 0;
      for (int t0 = tbeg; t0 < tend; t0 += 32) {
        const bool valid = t0 + lane < tend;
        const int w = wn;
        if (t0 + 32 < tend) wn = cand(t0 + 32 + lane);  // next chunk's load in flight
        const unsigned key = ((unsigned)(lane + 1) << 24) | (unsigned)w;
        unsigned h = hash_slot<HC>(w);
        unsigned old = valid ? (unsigned)atomicCAS(&hkey[h], -1, (int)key) : 0u;
        bool coll = valid && old != 0xffffffffu && (old & 0xffffffu) != (unsigned)w;
        if (__any_sync(FULL, coll)) {
          while (coll) {
            h = (h + 1) & (HC - 1);
            old = (unsigned)atomicCAS(&hkey[h], -1, (int)key);
            coll = old != 0xffffffffu && (old & 0xffffffu) != (unsigned)w;
          }
        }
        const bool mine = valid && (old == 0xffffffffu || (old >> 24) != 0u);
        if (mine && old != 0xffffffffu) atomicMin(reinterpret_cast<unsigned*>(&hkey[h]), key);
        __syncwarp();
        const bool isnew = mine && (unsigned)hkey[h] == key;
        __syncwarp();
        if (isnew) hkey[h] = w;
        const unsigned bal = __ballot_sync(FULL, isnew);
        if (isnew) lst[nl + __popc(bal & lt)] = w;
        nl += __popc(bal);
        if (nl > TH_LCAP) return false;
        __syncwarp();
      }
      return true;
    };
    ok = expand(0, Tsplit);
    const int nA = nl;
    // ---- X: the members of N(H) among s, N(s) and A, as ascending ranks
    int nx = 0;
    if (ok) {
      // s is a member (H is its neighbour); level 1 by the rows already located
      const bool m1 = lane < T0 && lane != hl && row_has(indices, pb, pd, H);
      const unsigned bm1 = __ballot_sync(FULL, m1);
      if (lane == 0) xs[0] = s;
      if (m1) xs[1 + __popc(bm1 & lt)] = w1;
      nx = 1 + __popc(bm1);  // <= 32
      for (int c0 = 0; c0 < nA && ok; c0 += 32) {
        const int c = c0 + lane;
        bool m = false;
        int x = 0;
        if (c < nA) {
          x = lst[c];
          const int bx = __ldg(indptr + x);
          m = row_has(indices, bx, __ldg(indptr + x + 1) - bx, H);
        }
        const unsigned bm = __ballot_sync(FULL, m);
        if (nx + __popc(bm) > TH_XCAP) {
          ok = false;
          break;
        }
        if (m) xs[nx + __popc(bm & lt)] = x;
        nx += __popc(bm);
      }
    }
    if (ok) {
      __syncwarp();
      int myrank = INT_MAX;
      for (int i0 = 0; i0 < nx; i0 += 4) {
        int xq[4], rq[4];
#pragma unroll
        for (int i = 0; i < 4; i++) xq[i] = xs[min(i0 + i, nx - 1)];
        hub_rank4(nh, D, xq, min(4, nx - i0), lane, rq);
#pragma unroll
        for (int i = 0; i < 4; i++)
          if (lane == i0 + i) myrank = rq[i];
      }
      int posx = 0;  // ascending order of the (distinct) ranks
      for (int i = 0; i < nx; i++) posx += __shfl_sync(FULL, myrank, i) < myrank;
      __syncwarp();
      if (lane < nx) xs[posx] = myrank;
      // ---- B: candidates new to the explicit ball, then minus N(H)
      ok = expand(Tsplit, Ts);
    }
    if (ok) {
      int kept = nA;
      for (int c0 = nA; c0 < nl; c0 += 32) {
        const int c = c0 + lane;
        bool keep = false;
        int x = 0;
        if (c < nl) {
          x = lst[c];
          const int bx = __ldg(indptr + x);
          keep = !row_has(indices, bx, __ldg(indptr + x + 1) - bx, H);
        }
        const unsigned bk = __ballot_sync(FULL, keep);
        __syncwarp();  // the chunk is read before it is overwritten
        if (keep) lst[kept + __popc(bk & lt)] = x;
        kept += __popc(bk);
      }
      nl = kept;
      __syncwarp();
    }
    if (!ok) {
      if (lane == 0) ovf_list[atomicAdd(ovf_count, 1)] = s;
      continue;
    }
    // ---- crossing level 2: n2 ids, r picks
    const int S = D - nx, n2 = nA + S + (nl - nA), r = K - T0;
    const unsigned long long fy_base = seed + SPLIT_GAMMA * (unsigned long long)(s + 1);
    int pos = lane;
    if (lane < r) {
      const unsigned long long z = splitmix_at(fy_base, lane);
      pos = lane + (n2 - lane <= 4096 ? umod64_tab(z, n2 - lane) : umod64_small(z, n2 - lane));
    }
    if (r > 1) pos = fy_positions(r, lane, pos, wsc);  // one pick: its draw is its position
    int v = 0;
    if (lane < r) {
      if (pos < nA) {
        v = lst[pos];
      } else if (pos < nA + S) {
        int q = pos - nA;
        for (int i = 0; i < nx && xs[i] <= q; i++) q++;
        v = __ldg(nh + q);
      } else {
        v = lst[pos - S];
      }
    }
    const int rk = rank_in_warp(r, v);
    if (lane < T0) {
      rn[lane] = w1;
      rd[lane] = 1;
    }
    if (lane < r) {
      rn[T0 + rk] = v;
      rd[T0 + rk] = 2;
    }
    if (lane == 0) out_cnt[item] = K;
    w_scanned += (unsigned long long)(T0 + Ts + D);
    w_expanded += (unsigned long long)(1 + T0);
    __syncwarp();
  }
  if (work && lane == 0) {
    atomicAdd(work, w_scanned);
    atomicAdd(work + 1, w_expanded);
  }
}

// ------------------------------------------------------------ tier C (CTA)
// Big balls (hub-adjacent sources of scale-free graphs: a level of thousands
// of ids): one CTA of 256 threads per source, the ball hash (HC slots), the
// discovered list and the level's parent ranges in shared memory.  A level is
// expanded 256 flattened entries at a time, one entry per thread; the parent
// of entry t comes from a bitmap of adjacency starts and per-word prefix
// counts.  First occurrences without MATCH: each entry inserts
// (t - t0 + 1) << 23 | id, equal ids keep the smallest tag (atomicMin), ids
// of earlier chunks and levels hold tag 0; after a barrier the entries whose
// slot holds their own key are the chunk's first occurrences, compacted in t
// order by warp ballots and a prefix over the 8 warp counts, and their slots
// retagged to 0.  Needs ids below 2^23 - 1; larger graphs keep the warp
// tier.  Replaces a 2-warp CTA with a 1024-id cap (12 warps per SM).
constexpr int TC_THREADS = 256, TC_HC = 4096, TC_CAP = 3072, TC_PCAP = 1024, TC_TCAP = 8192;
struct TierC {
  static constexpr int TW = TC_TCAP / 32;
  // hkey[HC] disc[CAP] ppre[PCAP] pbeg[PCAP] bmap[TW] pcnt[TW] jdraw[32] wcnt[8]
  static constexpr int WORDS = TC_HC + TC_CAP + 2 * TC_PCAP + 2 * TW + 32 + 8;
};

#ifndef TC_MINB
#define TC_MINB 5
#endif
__global__ void __launch_bounds__(TC_THREADS, TC_MINB)
    pbfs_cta(const int* __restrict__ indptr, const int* __restrict__ indices, int K,
             unsigned long long seed, long long src_begin, const int* __restrict__ list,
             const int* __restrict__ list_count, int* __restrict__ out_nbr,
             int* __restrict__ out_dist, int* __restrict__ out_cnt, int* __restrict__ ovf_list,
             int* __restrict__ ovf_count, int* __restrict__ queue,
             unsigned long long* __restrict__ work) {
  constexpr int HC = TC_HC, CAP = TC_CAP, PCAP = TC_PCAP, TCAP = TC_TCAP, TW = TierC::TW;
  __shared__ int s_it;
  constexpr unsigned EMPTY = 0xffffffffu, IDM = (1u << 23) - 1u;
  extern __shared__ __align__(16) int smem[];
  unsigned* const hkey = reinterpret_cast<unsigned*>(smem);
  int* const disc = smem + HC;
  int* const ppre = disc + CAP;
  int* const pbeg = ppre + PCAP;
  unsigned* const bmap = reinterpret_cast<unsigned*>(pbeg + PCAP);
  int* const pcnt = reinterpret_cast<int*>(bmap + TW);
  int* const jdraw = pcnt + TW;
  int* const wcnt = jdraw + 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt = (1u << lane) - 1u;
  unsigned long long w_scanned = 0, w_expanded = 0;
  // insert an id of a settled level (tag 0); true iff it was not there
  auto put0 = [&](int w) {
    unsigned h = hash_slot<HC>(w);
    for (;;) {
      const unsigned old = atomicCAS(&hkey[h], EMPTY, (unsigned)w);
      if (old == EMPTY || old == (unsigned)w) return;
      h = (h + 1) & (HC - 1);
    }
  };
  // block-wide exclusive prefix of one int per thread (+ total)
  auto block_scan = [&](int v, int& total) -> int {
    const int inc = warp_incl_scan(v);
    if (lane == 31) wcnt[warp] = inc;
    __syncthreads();
    int before = 0, tot = 0;
#pragma unroll
    for (int q = 0; q < TC_THREADS / 32; q++) {
      const int c = wcnt[q];
      before += q < warp ? c : 0;
      tot += c;
    }
    __syncthreads();
    total = tot;
    return before + inc - v;
  };
  const int total_items = *list_count;
  if (total_items == 0) return;  // (no storm of queue atomics for an empty list)
  // sources handed out one at a time (ball sizes, hence times, vary widely)
  for (;;) {
    if (tid == 0) s_it = atomicAdd(queue, 1);
    __syncthreads();
    const int it = s_it;
    if (it >= total_items) break;
    const int s = list[it];
    const long long item = (long long)s - src_begin;
    int* const rn = out_nbr + item * K;
    int* const rd = out_dist + item * K;
    const unsigned long long fy_base = seed + SPLIT_GAMMA * (unsigned long long)(s + 1);
    for (int i = tid; i < HC / 4; i += TC_THREADS)
      reinterpret_cast<uint4*>(hkey)[i] = make_uint4(EMPTY, EMPTY, EMPTY, EMPTY);
    const int b0 = __ldg(indptr + s);
    const int T0 = __ldg(indptr + s + 1) - b0;
    __syncthreads();
    bool ovf = T0 > CAP - 2;
    int count = 0, nst = 0, lb = 1, le = 1, depth = 1;
    if (!ovf) {
      // ---- level 1: the sorted adjacency of s
      if (tid == 0) put0(s);
      for (int t = tid; t < T0; t += TC_THREADS) {
        const int w = __ldg(indices + b0 + t);
        disc[1 + t] = w;
        put0(w);
      }
      w_scanned += tid == 0 ? (unsigned long long)T0 : 0ull;
      w_expanded += tid == 0 ? 1ull : 0ull;
      nst = T0;
      le = 1 + T0;
      __syncthreads();
    }
    // ---- levels: level `depth` is disc[lb, le) with nst ids; output it
    // (whole, or the Fisher-Yates subsample when it crosses K), expand it
    while (!ovf) {
      const int remaining = K - count;
      int take = nst;
      if (nst > remaining) {
        // crossing level: draws in parallel, the r swaps by one thread
        if (tid < remaining) jdraw[tid] = tid + umod64_tab(splitmix_at(fy_base, tid), nst - tid);
        __syncthreads();
        if (tid == 0) {
          for (int i = 0; i < remaining; i++) {
            const int j = jdraw[i];
            const int a = disc[le - nst + i];
            disc[le - nst + i] = disc[le - nst + j];
            disc[le - nst + j] = a;
          }
        }
        __syncthreads();
        take = remaining;
      }
      // rows: this level's picks ranked by id (levels come in distance order)
      if (tid < take) {
        const int v = disc[le - nst + tid];
        int r = 0;
        for (int q = 0; q < take; q++) r += disc[le - nst + q] < v;
        rn[count + r] = v;
        rd[count + r] = depth;
      }
      count += take;
      if (count >= K || nst == 0) break;
      // ---- expand: parents disc[lb, le) (nonzero degrees compacted)
      const int f = nst;
      if (f > PCAP) {
        ovf = true;
        break;
      }
      for (int w = tid; w < TW; w += TC_THREADS) bmap[w] = 0u;
      __syncthreads();
      int carry = 0, nne = 0;
      for (int i0 = 0; i0 < f; i0 += TC_THREADS) {
        const int i = i0 + tid;
        int d = 0, b = 0;
        if (i < f) {
          const int u = disc[lb + i];
          b = __ldg(indptr + u);
          d = __ldg(indptr + u + 1) - b;
        }
        // one scan for both prefixes: degree (low 22 bits; T > TCAP
        // overflows long before) and nonzero-degree rank (high bits)
        int ptot2;
        const int px = block_scan(d | (d > 0 ? 1 << 22 : 0), ptot2);
        const int dex = px & ((1 << 22) - 1), rex = px >> 22;
        const int dtot = ptot2 & ((1 << 22) - 1), ntot = ptot2 >> 22;
        if (d > 0) {
          const int r = nne + rex;
          const int p0 = carry + dex;
          ppre[r] = p0;
          pbeg[r] = b;
          if (p0 < TCAP) atomicOr(&bmap[p0 >> 5], 1u << (p0 & 31));
        }
        carry += dtot;
        nne += ntot;
      }
      const int T = carry;
      w_scanned += tid == 0 ? (unsigned long long)T : 0ull;
      w_expanded += tid == 0 ? (unsigned long long)f : 0ull;
      if (T > TCAP) {
        ovf = true;
        break;
      }
      __syncthreads();
      // prefix popcounts of the start bitmap (one word per thread)
      {
        const int nw = (T + 31) >> 5;  // words that hold entries
        if (nw <= 32) {
          if (warp == 0) {
            const int c = lane < nw ? __popc(bmap[lane]) : 0;
            pcnt[lane] = warp_incl_scan(c) - c;
          }
        } else {
          int ptot, pcarry = 0;
          for (int w0 = 0; w0 < nw; w0 += TC_THREADS) {
            const int w = w0 + tid;
            const int c = w < nw ? __popc(bmap[w]) : 0;
            const int ex = block_scan(c, ptot);
            if (w < nw) pcnt[w] = pcarry + ex;
            pcarry += ptot;
          }
        }
        __syncthreads();
      }
      lb = le;
      nst = 0;
      depth++;
      // entry t's id (0 past T); the next chunk's load is issued before this
      // chunk's hash work
      auto entry = [&](int t) -> int {
        if (t >= T) return 0;
        const int p = pcnt[t >> 5] + __popc(bmap[t >> 5] & ((2u << (t & 31)) - 1u)) - 1;
        return __ldg(indices + pbeg[p] + (t - ppre[p]));
      };
      int w_next = entry(tid);
      for (int t0 = 0; t0 < T; t0 += TC_THREADS) {
        const int t = t0 + tid;
        const bool valid = t < T;
        const int w = w_next;
        w_next = entry(t + TC_THREADS);
        const unsigned key = ((unsigned)(tid + 1) << 23) | (unsigned)w;
        unsigned h = hash_slot<HC>(w), old = 0u;
        if (valid) {
          for (;;) {
            old = atomicCAS(&hkey[h], EMPTY, key);
            if (old == EMPTY || (old & IDM) == (unsigned)w) break;
            h = (h + 1) & (HC - 1);
          }
        }
        const bool mine = valid && (old == EMPTY || (old >> 23) != 0u);
        if (mine && old != EMPTY) atomicMin(&hkey[h], key);
        __syncthreads();
        const bool isnew = mine && hkey[h] == key;
        const unsigned bal = __ballot_sync(FULL, isnew);
        if (lane == 0) wcnt[warp] = __popc(bal);
        __syncthreads();
        int before = 0, tot = 0;
#pragma unroll
        for (int q = 0; q < TC_THREADS / 32; q++) {
          const int c = wcnt[q];
          before += q < warp ? c : 0;
          tot += c;
        }
        if (isnew) {
          const int pos = le + nst + before + __popc(bal & lt);
          if (pos < CAP) disc[pos] = w;
          hkey[h] = (unsigned)w;  // settled: tag 0
        }
        nst += tot;
        __syncthreads();
        if (le + nst > CAP) {
          ovf = true;
          break;
        }
      }
      le += nst;
      __syncthreads();
    }
    if (ovf) {
      if (tid == 0) ovf_list[atomicAdd(ovf_count, 1)] = s;
    } else if (tid == 0) {
      out_cnt[item] = count;
    }
    __syncthreads();
  }
  if (work && tid == 0) {
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

#ifndef GU_LEAN_MINB
#define GU_LEAN_MINB 8
#endif
constexpr int T1A_CAP = 128, T1A_PCAP = 64, T1A_TCAP = 512, T1A_WARPS = 8;
constexpr int T1B_CAP = 1024, T1B_PCAP = 512, T1B_TCAP = 4096, T1B_WARPS = 2;

struct PbfsWs {
  int* ovfA;
  int* ovfB;
  int* ovf0;
  int* counts;  // [0]=ovfA count, [1]=ovfB count, [2]=ovf0 count, [3]=tier H rejects, [4]=F -> H directly, [5]=tier H work queue head, [6]=tier C work queue head
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
  size_t o0 = take(sizeof(int) * (size_t)(nsrc + 1));
  size_t oC = take(sizeof(int) * 8);
  size_t oW = take(sizeof(unsigned long long) * 2);
  size_t oS = take(sizeof(int) * 2 * (size_t)n * (size_t)slots);
  if (ws && base) {
    ws->ovfA = (int*)(base + oA);
    ws->ovfB = (int*)(base + oB);
    ws->ovf0 = (int*)(base + o0);
    ws->counts = (int*)(base + oC);
    ws->work = (unsigned long long*)(base + oW);
    ws->slots = (int*)(base + oS);
  }
  return off;
}

constexpr int TF_WARPS = 8;

cudaError_t launch_fast(int sms, long long n, const int* indptr, const int* indices, int k,
                        unsigned long long seed, long long src_begin, long long nsrc,
                        int* out_nbr, int* out_dist, int* out_count, int* ovf_out, int* ovf_cnt,
                        int* hub_out, int* hub_cnt, int* hub_direct, unsigned long long* work,
                        cudaStream_t st) {
  // packed tags need ids below 2^24 - 1 (the empty key is all ones)
  auto kern = n < (1 << 24) - 1 ? pbfs_fast<TF_WARPS, true> : pbfs_fast<TF_WARPS, false>;
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TF_WARPS * 32, 0);
  if (e != cudaSuccess) return e;
  long long blocks = (nsrc + TF_WARPS - 1) / TF_WARPS;
  long long cap = (long long)sms * (per_sm > 0 ? per_sm : 1) * 8;
  if (blocks > cap) blocks = cap;
  kern<<<(unsigned)blocks, TF_WARPS * 32, 0, st>>>(indptr, indices, k, seed, src_begin, nsrc,
                                                   out_nbr, out_dist, out_count, ovf_out, ovf_cnt,
                                                   hub_out, hub_cnt, hub_direct, work);
  return cudaGetLastError();
}

template <int CAP, int PCAP, int TCAP, int W, int MINB>
cudaError_t launch_warp_tier(int sms, long long n, const int* indptr, const int* indices, int k,
                             unsigned long long seed, long long src_begin, long long nsrc,
                             const int* list, const int* list_count, int* out_nbr, int* out_dist,
                             int* out_count, int* ovf_out, int* ovf_cnt, unsigned long long* work,
                             cudaStream_t st) {
  using LA = Tier1<32, CAP, PCAP, TCAP>;
  constexpr size_t smem = sizeof(int) * LA::WORDS * W;
  auto kern = n < (1 << 24) - 1 ? pbfs_warp<CAP, PCAP, TCAP, W, MINB, true>
                                : pbfs_warp<CAP, PCAP, TCAP, W, MINB, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, W * 32, smem);
  if (e != cudaSuccess) return e;
  long long blocks = (nsrc + W - 1) / W;
  long long cap = (long long)sms * (per_sm > 0 ? per_sm : 1) * (list ? 1 : 8);
  if (blocks > cap) blocks = cap;
  kern<<<(unsigned)blocks, W * 32, smem, st>>>(indptr, indices, k, seed, src_begin, nsrc, list,
                                                list_count, out_nbr, out_dist, out_count, ovf_out,
                                                ovf_cnt, work);
  return cudaGetLastError();
}

// tier 1a: lean warp, CAP 128
cudaError_t launch_lean(int sms, long long n, const int* indptr, const int* indices, int k,
                        unsigned long long seed, long long src_begin, long long nsrc,
                        const int* list, const int* list_count, int* out_nbr, int* out_dist,
                        int* out_count, int* ovf_out, int* ovf_cnt, unsigned long long* work,
                        cudaStream_t st) {
  return launch_warp_tier<T1A_CAP, T1A_PCAP, T1A_TCAP, 8, GU_LEAN_MINB>(
      sms, n, indptr, indices, k, seed, src_begin, nsrc, list, list_count, out_nbr, out_dist, out_count,
      ovf_out, ovf_cnt, work, st);
}

// tier 1b: the same lean warp kernel with CAP 1024 (hub-adjacent balls)
cudaError_t launch_lean_big(int sms, long long n, const int* indptr, const int* indices, int k,
                            unsigned long long seed, long long src_begin, long long nsrc,
                            const int* list, const int* list_count, int* out_nbr, int* out_dist,
                            int* out_count, int* ovf_out, int* ovf_cnt, unsigned long long* work,
                            cudaStream_t st) {
  return launch_warp_tier<T1B_CAP, T1B_PCAP, T1B_TCAP, 2, 1>(
      sms, n, indptr, indices, k, seed, src_begin, nsrc, list, list_count, out_nbr, out_dist, out_count,
      ovf_out, ovf_cnt, work, st);
}

// tier H: hub-adjacent sources of the list, one warp each (ids below 2^24 - 1)
cudaError_t launch_hub(int sms, const int* indptr, const int* indices, int k,
                       unsigned long long seed, long long src_begin, const int* list,
                       const int* list_count, int* out_nbr, int* out_dist, int* out_count,
                       int* ovf_out, int* ovf_cnt, int* queue, unsigned long long* work,
                       cudaStream_t st) {
  constexpr size_t smem = sizeof(int) * TierH::WORDS * TH_WARPS;
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pbfs_hub, TH_WARPS * 32, smem);
  if (e != cudaSuccess) return e;
  const unsigned blocks = (unsigned)sms * (unsigned)(per_sm > 0 ? per_sm : 1);
  pbfs_hub<<<blocks, TH_WARPS * 32, smem, st>>>(indptr, indices, k, seed, src_begin, list, list_count,
                                                out_nbr, out_dist, out_count, ovf_out, ovf_cnt, queue,
                                                work);
  return cudaGetLastError();
}

// tier C: one 256-thread CTA per big-ball source (ids below 2^23 - 1)
cudaError_t launch_cta(int sms, const int* indptr, const int* indices, int k,
                       unsigned long long seed, long long src_begin, const int* list,
                       const int* list_count, int* out_nbr, int* out_dist, int* out_count,
                       int* ovf_out, int* ovf_cnt, int* queue, unsigned long long* work,
                       cudaStream_t st) {
  constexpr size_t smem = sizeof(int) * TierC::WORDS;
  cudaError_t e = cudaFuncSetAttribute(pbfs_cta, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pbfs_cta, TC_THREADS, smem);
  if (e != cudaSuccess) return e;
  const unsigned blocks = (unsigned)sms * (unsigned)(per_sm > 0 ? per_sm : 1);
  pbfs_cta<<<blocks, TC_THREADS, smem, st>>>(indptr, indices, k, seed, src_begin, list, list_count,
                                              out_nbr, out_dist, out_count, ovf_out, ovf_cnt, queue,
                                              work);
  return cudaGetLastError();
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
  GU_CHECK(cudaMemsetAsync(ws.counts, 0, 8 * sizeof(int), st));
  if (k == 0) {
    GU_CHECK(cudaMemsetAsync(out_count, 0, sizeof(int32_t) * nsrc, st));
    return GU_OK;
  }
  const int sms = sm_count();
  if (k <= 32) {
    // tier F (register fast path) -> tier 1a (lean warp per source, CAP 128)
    // -> tier 1b (CAP 1024) -> tier 2.  GU_PBFS_MODE=lean skips tier F
    // (comparison only; every path is exact).
    static const char* env_mode = getenv("GU_PBFS_MODE");
    // tier H (hub-adjacent sources) needs ids below 2^24 - 1; GU_PBFS_HUB=0
    // skips it (comparison only)
    static const char* env_hub = getenv("GU_PBFS_HUB");
    const bool use_hub = n < (1 << 24) - 1 && !(env_hub && !strcmp(env_hub, "0"));
    if (!env_mode || strcmp(env_mode, "lean")) {
      GU_CHECK(launch_fast(sms, n, indptr, indices, k, seed, src_begin, nsrc, out_nbr, out_dist,
                           out_count, ws.ovf0, ws.counts + 2, use_hub ? ws.ovfA : nullptr,
                           ws.counts + 0, ws.counts + 4, work, st));
      GU_CHECK(launch_lean(sms, n, indptr, indices, k, seed, src_begin, nsrc, ws.ovf0, ws.counts + 2,
                           out_nbr, out_dist, out_count, ws.ovfA, ws.counts + 0, work, st));
    } else {
      GU_CHECK(launch_lean(sms, n, indptr, indices, k, seed, src_begin, nsrc, nullptr, nullptr,
                           out_nbr, out_dist, out_count, ws.ovfA, ws.counts + 0, work, st));
    }
    // hub-adjacent sources (tier H): tier 1a's overflow and tier F's direct
    // hand-offs; what it cannot take goes on to the big-ball tiers.  Its
    // reject list borrows ovf0 (tier 1a has consumed it) and counts[3].
    const int* big_list = ws.ovfA;
    const int* big_count = ws.counts + 0;
    if (use_hub) {
      GU_CHECK(launch_hub(sms, indptr, indices, k, seed, src_begin, ws.ovfA, ws.counts + 0, out_nbr,
                          out_dist, out_count, ws.ovf0, ws.counts + 3, ws.counts + 5, work, st));
      big_list = ws.ovf0;
      big_count = ws.counts + 3;
    } else {
      GU_CHECK(cudaMemcpyAsync(ws.counts + 3, ws.counts + 0, sizeof(int), cudaMemcpyDeviceToDevice, st));
    }
    // big balls: the CTA tier when ids fit its 23-bit packed keys
    static const char* env_big = getenv("GU_PBFS_BIG");
    if (n < (1 << 23) - 1 && !(env_big && !strcmp(env_big, "warp"))) {
      GU_CHECK(launch_cta(sms, indptr, indices, k, seed, src_begin, big_list, big_count, out_nbr,
                          out_dist, out_count, ws.ovfB, ws.counts + 1, ws.counts + 6, work, st));
    } else {
      GU_CHECK(launch_lean_big(sms, n, indptr, indices, k, seed, src_begin, nsrc, big_list, big_count,
                               out_nbr, out_dist, out_count, ws.ovfB, ws.counts + 1, work, st));
    }
  } else {
    // k > group size: every source goes straight to the exact tier-2 path
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

extern "C" int gu_partial_bfs_tier_counts(void* workspace, int64_t nsrc, int32_t* host_out4) {
  PbfsWs ws;
  pbfs_ws_layout(1, nsrc, 1, (char*)workspace, &ws);
  int c[5];
  GU_CHECK(cudaMemcpy(c, ws.counts, 5 * sizeof(int), cudaMemcpyDeviceToHost));
  host_out4[0] = c[2] + c[4];  // left tier F (to tier 1a, or straight to tier H)
  host_out4[1] = c[0];         // entered tier H (from tier 1a or tier F)
  host_out4[2] = c[3];         // entered tier C / 1b
  host_out4[3] = c[1];         // entered tier 2
  return GU_OK;
}

extern "C" int gu_partial_bfs_overflow_counts(void* workspace, int64_t nsrc, int32_t* host_out3) {
  PbfsWs ws;
  pbfs_ws_layout(1, nsrc, 1, (char*)workspace, &ws);
  int c[5];
  GU_CHECK(cudaMemcpy(c, ws.counts, 5 * sizeof(int), cudaMemcpyDeviceToHost));
  host_out3[0] = c[2] + c[4];  // left tier F
  host_out3[1] = c[3];         // reached the big-ball tier (C / 1b)
  host_out3[2] = c[1];         // reached tier 2
  return GU_OK;
}
