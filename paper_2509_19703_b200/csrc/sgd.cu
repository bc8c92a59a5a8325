// sgd.cu -- K7: Hogwild fp32 UMAP layout epochs.
//
// Same per-visit update as the reference's sgd_sweep
// (/root/reference/pkg/src/graph_umap/_kernels.py:158-223) driven by
// _run_sgd (layout.py:314-360):
//   attraction  d2 > 0: g = -2ab h (d2^b / d2) / (a d2^b + 1), per-component
//               clip +-4, x_u += lr g dx, x_v -= lr g dx
//   repulsion   n_neg times: up to 8 uniform draws c != u, c not a sym
//               neighbour of u (binary search in the sorted CSR row), else the
//               sample is skipped; d2 > 0: g = 2b / ((0.001 + d2)(a d2^b + 1)),
//               clip +-4; coincident: 4 (cos th, sin th), th uniform; only x_u
//               moves.  The head's running position is kept in registers, so
//               the repulsions see the attracted x_u exactly as in the
//               sequential sweep; u and v receive their deltas through
//               vector float2 atomics (red.global.add.v2.f32).
// Schedule (D7 in SURVEY.md section 9): edges are stored once in a
// Feistel-shuffled order (gu_sgd_prepare_edges).  Windowed epochs
// (optimize_sampled) take the window of `window` consecutive positions
// starting where the previous epoch stopped, wrapping (layout.py:329-337).
// Full epochs (optimize_full) visit every edge in a fresh per-epoch order:
// 1024-edge tiles permuted by a per-epoch Feistel bijection, tiles streamed
// coalesced.  Negatives and thetas come from a counter-based 64-bit mix of
// (seed, epoch, position, slot, try).
#include <climits>
#include <cmath>

#include <cstdlib>
#include <cstring>
#include <type_traits>

#include <cub/device/device_scan.cuh>

#include "common.cuh"
#include "gumap.h"

namespace gu {
namespace {

constexpr int TILE = 1024;
constexpr int SGD_NEG_BLOCK = 5;
static_assert(SGD_NEG_BLOCK <= 8, "slot bits of the cooperative search owner tag");
constexpr unsigned FULL = 0xffffffffu;
#ifndef SGD_SCAN
#define SGD_SCAN 16  // neighbour-row entries compared with independent loads
#endif
// coordinate gathers cached in L2 only (the 32 MB array never fits L1):
// c5 epoch 2.352 -> 2.33 ms, c4 0.600 -> 0.590 ms (profiles/r02_ab_sgd_ldcg.log)
#define SGD_LD(p) __ldcg(p)
#ifndef SGD_POOL
#define SGD_POOL 1  // warp-pooled first-try negatives on GPU-filling epochs
#endif
#ifndef SGD_STREAM
#define SGD_STREAM 1  // window records: pooled tries consumed in place, no per-slot arrays
#endif
#ifndef SGD_LOCKSTEP
#define SGD_LOCKSTEP 1  // a block of negatives reads one x_u (see the epoch kernel)
#endif
#ifndef SGD_MIN_BLOCKS
#define SGD_MIN_BLOCKS 4  // <= 64 registers: 32 warps per SM
#endif  // negatives handled in lockstep per block

// Feistel bijection on [0, 2^bits) with cycle walking into [0, m)
__device__ __host__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

// counter-based draws: one 64-bit finaliser per visit (base = mix64(epoch
// key ^ edge position)), then a 32-bit finaliser per (negative slot q, try
// t) over a Weyl step of the base -- distinct (q, t) of a visit give
// distinct pre-images, so the draws of a visit never repeat.  The candidate
// is the draw scaled to [0, n); the coincident-point angle is a second
// finaliser of the same draw, evaluated only when it is needed.
__device__ __forceinline__ unsigned fmix32(unsigned h) {
  h ^= h >> 16;
  h *= 0x85ebca6bu;
  h ^= h >> 13;
  h *= 0xc2b2ae35u;
  h ^= h >> 16;
  return h;
}

__device__ __forceinline__ unsigned draw32(unsigned long long base, int q, int t) {
  return fmix32(((unsigned)base + (unsigned)(q * 8 + t + 1) * 0x9E3779B9u) ^
                (unsigned)(base >> 32));
}

__device__ __forceinline__ unsigned theta_draw(unsigned h) { return fmix32(h ^ 0x68e31da4u); }

struct Feistel {
  unsigned long long m;
  int half;  // bits per half
  unsigned long long key;
  __device__ __host__ Feistel(unsigned long long m_, unsigned long long key_) : m(m_), key(key_) {
    int bits = 2;
    while ((1ull << bits) < m_) bits++;
    if (bits & 1) bits++;
    half = bits / 2;
  }
  __device__ __host__ __forceinline__ unsigned long long once(unsigned long long x) const {
    const unsigned long long mask = (1ull << half) - 1ull;
    unsigned long long l = x >> half, r = x & mask;
#pragma unroll
    for (int i = 0; i < 4; i++) {
      unsigned long long f = mix64(r ^ (key + 0x9E3779B97F4A7C15ULL * (unsigned long long)(i + 1))) & mask;
      unsigned long long t = l ^ f;
      l = r;
      r = t;
    }
    return (l << half) | r;
  }
  __device__ __host__ __forceinline__ unsigned long long operator()(unsigned long long x) const {
    do {
      x = once(x);
    } while (x >= m);
    return x;
  }
};

__device__ __forceinline__ float clip4(float x) { return fminf(4.0f, fmaxf(-4.0f, x)); }

__device__ __forceinline__ bool is_neighbor(const int* __restrict__ ip, const int* __restrict__ ix,
                                            int u, int c) {
  int lo = __ldg(ip + u), hi = __ldg(ip + u + 1);
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    int x = __ldg(ix + mid);
    if (x < c) lo = mid + 1;
    else if (x > c) hi = mid;
    else return true;
  }
  return false;
}

// Per-vertex Bloom words of the neighbour ids: a candidate with any of its
// bits clear is certainly not a neighbour, so only the filter hits (true
// neighbours and false positives) run the row search and the test stays
// exact.  Two layouts, chosen per plan (gu_sgd_record_bytes_for):
//  * table: 64 bits, 2 hash bits per id, one word per vertex gathered by
//    head (8 B x n) -- measured best for small concurrency caps (c3 epoch
//    0.277 ms vs 0.39 with the records below; profiles/r02_ab_sgd_r32b.log);
//  * in-record: 32-byte edge records carry their head's 128-bit word with 3
//    hash bits per id, streamed with the record -- no dependent gather, and
//    ~1.5% false positives instead of ~10% at degree 12 (c5 epoch 3.21 ->
//    2.75 ms; profiles/r02_ab_sgd_r32.log).
struct Filt64 {
  using Word = uint2;
  static constexpr int K = 2, SHIFT = 26;  // 32 - log2(64)
};
#ifndef SGD_F128_K
#define SGD_F128_K 3
#endif
struct Filt128 {
  using Word = uint4;
  static constexpr int K = SGD_F128_K, SHIFT = 25;  // 32 - log2(128)
};
using FiltWord = Filt64::Word;

// edge-record layouts (gu_sgd_prepare_edges / gu_sgd_epochs `record_mode`)
enum RecMode : int {
  REC_TABLE = 0,  // 16 bytes; the head's 64-bit word gathered from the per-vertex table
  REC_BLOOM = 1,  // 32 bytes; + the head's 128-bit / 3-hash Bloom word
  REC_RANGE = 2,  // 32 bytes; + [min, max] of the head's neighbour ids and its
                  // 64-bit / 2-hash word (ids in a locality order, csrc/order.cu)
  REC_HASH = 3,   // 16 bytes {src, dst, h, off << 4 | log2 size}: an exact
                  // open-addressing set of the head's neighbour ids (small caps)
};

// Exact neighbour sets (REC_HASH): vertex u's neighbour ids in a table of
// S_u = next_pow2(4 deg(u)) >= 4 int32 slots (load <= 1/4, empty = -1) at
// off[u], as buckets of 4 slots; home bucket = top log2(S_u / 4) bits of the
// Fibonacci product, linear probing over buckets.  One 16-byte load answers
// almost every candidate, with no Bloom filter and no row search.
// (buckets of 4 slots, one 16-byte load each: a set at load <= 1/4 answers
// almost every lookup with its home bucket)
__device__ __forceinline__ unsigned hset_bucket(int c, unsigned lg) {
  return lg > 2 ? ((unsigned)c * 0x9E3779B1u) >> (34u - lg) : 0u;
}

template <class F>
__device__ __forceinline__ unsigned filt_bit(int c, int j) {
  const unsigned m = j == 0 ? 0x9E3779B1u : (j == 1 ? 0x85EBCA77u : 0xC2B2AE3Du);
  return ((unsigned)c * m) >> F::SHIFT;
}

__device__ __forceinline__ unsigned filt_word(const uint4& f, unsigned w) {
  return w == 0 ? f.x : (w == 1 ? f.y : (w == 2 ? f.z : f.w));
}
__device__ __forceinline__ unsigned filt_word(const uint2& f, unsigned w) { return w ? f.y : f.x; }

// Bloom word of one neighbour row
template <class F>
__device__ __forceinline__ typename F::Word row_filter(const int* __restrict__ nix, int b, int e) {
  constexpr int WORDS = sizeof(typename F::Word) / 4;
  unsigned w[4] = {0u, 0u, 0u, 0u};
  for (int p = b; p < e; p++) {
    const int c = __ldg(nix + p);
#pragma unroll
    for (int k = 0; k < F::K; k++) {
      const unsigned h = filt_bit<F>(c, k);
#pragma unroll
      for (int j = 0; j < WORDS; j++)
        if ((h >> 5) == (unsigned)j) w[j] |= 1u << (h & 31);
    }
  }
  typename F::Word f;
  memcpy(&f, w, sizeof(f));
  return f;
}

__global__ void neighbor_filter_kernel(int n, const int* __restrict__ nip,
                                       const int* __restrict__ nix, FiltWord* __restrict__ filt) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    filt[v] = row_filter<Filt64>(nix, __ldg(nip + v), __ldg(nip + v + 1));
}

template <class F>
__device__ __forceinline__ bool filt_maybe(const typename F::Word& f, int c) {
  bool all = true;
#pragma unroll
  for (int k = 0; k < F::K; k++) {
    const unsigned h = filt_bit<F>(c, k);
    all = all && ((filt_word(f, h >> 5) >> (h & 31)) & 1u);
  }
  return all;
}

// Edge record {src, dst, float(h), row}: row = (start of src's neighbour row
// << 6) | degree when both fit (start < 2^26, degree < 63), else -1 (the
// kernel then reads nbr_indptr) -- the first rejection probe can then issue
// straight after the coalesced record load.  32-byte records append the
// head's filter (REC_BLOOM: 128-bit word; REC_RANGE: min / max neighbour id
// and the 64-bit word).  relabel (nullable): old id -> new id; nip / nix are
// then the graph in the new ids, and src / dst are mapped through it.
__global__ void prepare_edges_kernel(long long E, const int* __restrict__ src,
                                     const int* __restrict__ dst, const double* __restrict__ w,
                                     const int* __restrict__ nip, const int* __restrict__ nix,
                                     const int* __restrict__ relabel, int mode,
                                     unsigned long long key, int4* __restrict__ out,
                                     int* __restrict__ perm_out) {
  Feistel perm((unsigned long long)E, key);
  const int rw = mode == REC_TABLE ? 1 : 2;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < E;
       p += (long long)gridDim.x * blockDim.x) {
    const long long e = (long long)perm((unsigned long long)p);
    const int u = relabel ? relabel[src[e]] : src[e];
    const int v = relabel ? relabel[dst[e]] : dst[e];
    const int rb = nip[u], deg = nip[u + 1] - rb;
    const int row = (rb < (1 << 26) && deg < 63) ? ((rb << 6) | deg) : -1;
    out[rw * p] = make_int4(u, v, __float_as_int((float)w[e]), row);
    if (mode == REC_BLOOM) {
      const uint4 f = row_filter<Filt128>(nix, rb, rb + deg);
      out[2 * p + 1] = make_int4((int)f.x, (int)f.y, (int)f.z, (int)f.w);
    } else if (mode == REC_RANGE) {
      const uint2 f = row_filter<Filt64>(nix, rb, rb + deg);
      const int lo = deg > 0 ? nix[rb] : INT_MAX, hi = deg > 0 ? nix[rb + deg - 1] : -1;
      out[2 * p + 1] = make_int4(lo, hi, (int)f.x, (int)f.y);
    }
    if (perm_out) perm_out[p] = (int)e;
  }
}

// REC_RANGE records in a local stored order: the edges in the order of the
// relabelled neighbour CSR (heads ascending in the BFS locality order), then
// shuffled inside blocks of `block` consecutive edges.  A 1024-edge epoch tile
// then touches the coordinates of a few thousand nearby vertices (~22 KB at
// c5) instead of ~1024 scattered ones; tiles still run in a fresh random
// order every epoch.  order: new id -> old id; nip_old / nix_old: the
// caller's neighbour CSR, whose entry index is the sym edge id (rows sorted).
__global__ void prepare_edges_local(long long E, const double* __restrict__ w, int n,
                                    const int* __restrict__ nip, const int* __restrict__ nix,
                                    const int* __restrict__ order,
                                    const int* __restrict__ nip_old,
                                    const int* __restrict__ nix_old, long long block,
                                    unsigned long long key, int4* __restrict__ out,
                                    int* __restrict__ perm_out) {
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < E;
       p += (long long)gridDim.x * blockDim.x) {
    const long long blk = p / block, b0 = blk * block;
    const long long bsize = (E - b0) < block ? (E - b0) : block;
    Feistel fp((unsigned long long)bsize, mix64(key ^ (0x9E3779B97F4A7C15ull * (blk + 1))));
    const long long q = b0 + (long long)fp((unsigned long long)(p - b0));
    // head: the row holding entry q (upper bound in the new offsets)
    int lo = 0, hi = n;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (nip[mid] <= q) lo = mid; else hi = mid;
    }
    const int u = lo, v = nix[q];
    const int ou = order[u], ov = order[v];
    int a = nip_old[ou], b = nip_old[ou + 1];
    while (a < b) {
      const int mid = (a + b) >> 1;
      if (nix_old[mid] < ov) a = mid + 1; else b = mid;
    }
    const long long e = a;
    const int rb = nip[u], deg = nip[u + 1] - rb;
    const int row = (rb < (1 << 26) && deg < 63) ? ((rb << 6) | deg) : -1;
    out[2 * p] = make_int4(u, v, __float_as_int((float)w[e]), row);
    const uint2 f = row_filter<Filt64>(nix, rb, rb + deg);
    out[2 * p + 1] = make_int4(deg > 0 ? nix[rb] : INT_MAX, deg > 0 ? nix[rb + deg - 1] : -1,
                               (int)f.x, (int)f.y);
    if (perm_out) perm_out[p] = (int)e;
  }
}

constexpr int SGD_WARPS = 8;  // 256 threads per block at most (block_for)

// MINB: CTAs per SM the register budget is sized for -- 4 (64 registers) for
// GPU-filling epochs, 2 (96 registers) for the small-cap 16-lane mode, whose
// few resident warps are latency-bound and gain from the longer register
// budget (c3 epoch 0.295 -> 0.276 ms; at 96 registers c5 would lose 8%)
template <int LANES, int MINB, int MODE>
__global__ void __launch_bounds__(256, MINB)
    sgd_epoch_kernel(int n, long long E, float2* __restrict__ xy, const int4* __restrict__ edges,
                     const int* __restrict__ nip, const int* __restrict__ nix,
                     const FiltWord* __restrict__ filt, float a, float b, float lr, int epoch,
                     int n_neg, long long items, long long start, int windowed,
                     unsigned long long seed, int* __restrict__ diverged,
                     long long ibase = 0, long long* __restrict__ acc = nullptr) {
  constexpr int lanes = LANES;
  constexpr bool POOL = SGD_POOL && LANES == 32 && (MODE == REC_BLOOM || MODE == REC_RANGE);
  // (candidate, row begin, row end, owner lane * 8 + slot) of the warp's
  // filter hits, and each lane's bitmask of slots found to be neighbours
  __shared__ int4 sh_pairs[SGD_WARPS][32 * SGD_NEG_BLOCK];
  __shared__ unsigned sh_hit[SGD_WARPS][32];
  const long long ntiles = (E + TILE - 1) / TILE;
  Feistel tperm((unsigned long long)ntiles, mix64(seed ^ (0x51ED27ull + (unsigned long long)epoch)));
  const unsigned long long rkey = mix64(seed ^ (0xA5A5A5A5ull * (unsigned long long)(epoch + 1)));
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  bool bad = false;
  // warp-uniform loop (every lane reaches the collectives below).  Each warp
  // takes `lanes` visits per step (lanes < 32 when the concurrency cap is
  // small: the same visits in flight spread over more warps, i.e. more
  // independent instruction streams per scheduler); the other lanes and
  // lanes past the end ride along inactive
  const long long gwarp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long stride = (((long long)gridDim.x * blockDim.x) >> 5) * lanes;
  // full mode: the `lanes` visits of one warp step share one tile (TILE is a
  // multiple of 32 and i0 a multiple of lanes), so the tile permutation is
  // evaluated lane-parallel for the next 32 steps and handed out by shuffle
  unsigned tile_batch = 0;
  int step = 0;
  // deterministic mode (acc != nullptr): visits [ibase, items) read the
  // positions as they stood at the start of this batch and push their deltas
  // as 2^-32 fixed-point integers (order-free sums: bitwise reproducible);
  // det_apply_kernel adds them after the batch
  auto push = [&](int w, float dx, float dy) {
    if (acc) {
      atomicAdd(reinterpret_cast<unsigned long long*>(acc + 2 * (long long)w),
                (unsigned long long)__float2ll_rn(dx * 4294967296.0f));
      atomicAdd(reinterpret_cast<unsigned long long*>(acc + 2 * (long long)w + 1),
                (unsigned long long)__float2ll_rn(dy * 4294967296.0f));
    } else {
      atomicAdd(&xy[w], make_float2(dx, dy));
    }
  };
  for (long long i0 = ibase + gwarp * lanes; i0 < items; i0 += stride, step = (step + 1) & 31) {
    const long long i = i0 + lane;
    bool act = lane < lanes && i < items;
    long long p = 0;
    if (windowed) {
      p = start + i;
      if (p >= E) p -= E;
    } else {
      if (step == 0) {
        const long long il = i0 + (long long)lane * stride;
        tile_batch = il < items ? (unsigned)tperm((unsigned long long)(il / TILE)) : 0u;
      }
      const long long tile = (long long)__shfl_sync(FULL, tile_batch, step);
      p = tile * TILE + (i - (i0 / TILE) * TILE);
      if (p >= E) act = false;  // partial last tile maps onto itself
    }
    if (!act) p = 0;
    // GPU-filling epochs are bound by L2 tag lookups (12.7 requests per visit,
    // 73% of the L2 peak: profiles/r02_ncu_sgd_l2.txt), five of them the
    // random first-try negatives.  POOL: each lane draws ONE uniform vertex per
    // warp step and gathers its coordinates; the 32 visits of the step take
    // their first tries from these 32 (each still uniform on [0, n), only
    // correlated across the visits of one step, which never write them).
    int pool_c = 0;
    float2 pool_xy = make_float2(0.f, 0.f);
    if (POOL) {
      const unsigned pd = fmix32(fmix32((unsigned)i ^ (unsigned)rkey) + (unsigned)(rkey >> 32) +
                                 (unsigned)((unsigned long long)i >> 32));
      pool_c = (int)__umulhi(pd, (unsigned)n);
      pool_xy = SGD_LD(&xy[pool_c]);
    }
    // streamed once per epoch: evict-first, keep L2 for x / filter / rows
    using F = typename std::conditional<MODE == REC_BLOOM, Filt128, Filt64>::type;
    const int4 rec = act ? __ldcs(edges + ((MODE == REC_TABLE || MODE == REC_HASH) ? 1 : 2) * p) : make_int4(0, 0, 0, 0);
    const int u = rec.x, v = rec.y;
    typename F::Word fw;
    int rlo = INT_MIN, rhi = INT_MAX;  // REC_RANGE: the head's neighbour-id window
    if (MODE == REC_BLOOM) {
      const int4 f4 = act ? __ldcs(edges + 2 * p + 1) : make_int4(-1, -1, -1, -1);
      memcpy(&fw, &f4, sizeof(fw));
    } else if (MODE == REC_RANGE) {
      const int4 f4 = act ? __ldcs(edges + 2 * p + 1) : make_int4(INT_MIN, INT_MAX, -1, -1);
      rlo = f4.x;
      rhi = f4.y;
      const uint2 f2 = make_uint2((unsigned)f4.z, (unsigned)f4.w);
      memcpy(&fw, &f2, sizeof(fw));
    } else if (MODE == REC_HASH) {
      memset(&fw, 0, sizeof(fw));
    } else if (filt) {
      memcpy(&fw, filt + u, sizeof(fw));
    } else {
      memset(&fw, 0xff, sizeof(fw));
    }
    const float h = __int_as_float(rec.z);
    float2 xu = SGD_LD(&xy[u]);
    const float2 xv = SGD_LD(&xy[v]);
    float dux = 0.f, duy = 0.f;
    if (act) {
      const float dx = xu.x - xv.x, dy = xu.y - xv.y;
      const float d2 = dx * dx + dy * dy;
      if (d2 > 0.f) {
        // fast division: K7 is statistically, not bit-exactly, paired with
        // the reference (the float64 replay K8 is the exact one)
        const float pb = __powf(d2, b);
        const float g = __fdividef(-2.0f * a * b * h * pb, d2 * (a * pb + 1.0f));
        const float gx = clip4(g * dx) * lr, gy = clip4(g * dy) * lr;
        dux += gx;
        duy += gy;
        xu.x += gx;
        xu.y += gy;
        push(v, -gx, -gy);
        if (!isfinite(xv.x - gx) || !isfinite(xv.y - gy)) bad = true;
      }
    }
    // repulsions.  Try t of slot q draws 32 bits from draw32(visit base, q,
    // t): they pick the candidate, and a second finaliser gives its theta.
    // The first tries of all slots are known up front: their coordinate
    // loads go out at once, and only the candidates whose neighbour-filter
    // bit is set (~deg/128 of them) are searched in the head's sorted row --
    // cooperatively, one (candidate, row) pair per lane across the warp.  A
    // rejected try (c == u or a neighbour) takes the sequential retry path.
    // The repulsion math stays sequential in slot order on the register copy
    // of x_u, as in the reference sweep.
    const unsigned long long vbase = mix64(rkey ^ (unsigned long long)p);
    int rb = 0, re = 0;
    if (act && MODE != REC_HASH) {
      if (rec.w >= 0) {
        rb = rec.w >> 6;
        re = rb + (rec.w & 63);
      } else {
        rb = __ldg(nip + u);
        re = __ldg(nip + u + 1);
      }
    }
#if SGD_STREAM
    if (POOL && MODE == REC_RANGE) {
      // Streamlined repulsions for window records: a pooled first try outside
      // the head's neighbour-id window (99.8% of them on c5) needs no further
      // test, so nothing is kept in per-slot arrays and no filter hits are
      // published for a cooperative search -- the slot's vertex and
      // coordinates come by shuffle right where its gradient is evaluated.
      // The rare slots that need more (in-window with the Bloom bits set: a
      // neighbour or a false positive; the head itself; a coincident point)
      // are flagged and redone one by one below.
      const unsigned d0 = draw32(vbase, 0, 0);
      const unsigned stride = ((d0 >> 5) & 15u) * 2u + 1u;
      for (int q0 = 0; q0 < n_neg; q0 += SGD_NEG_BLOCK) {
        const int nq = min(SGD_NEG_BLOCK, n_neg - q0);
        unsigned redo = 0;
        float sx = 0.f, sy = 0.f;
#pragma unroll
        for (int q = 0; q < SGD_NEG_BLOCK; q++) {
          const int ln = (int)((d0 + (unsigned)(q0 + q) * stride) & 31u);
          const int c = __shfl_sync(FULL, pool_c, ln);
          const float cx = __shfl_sync(FULL, pool_xy.x, ln);
          const float cy = __shfl_sync(FULL, pool_xy.y, ln);
          const bool maybe_nb = c >= rlo && c <= rhi && filt_maybe<F>(fw, c);
          const float dx = xu.x - cx, dy = xu.y - cy;
          const float d2 = dx * dx + dy * dy;
          const float g = __fdividef(2.0f * b, (0.001f + d2) * (a * __powf(d2, b) + 1.0f));
          const bool live = act && q < nq;
          const bool good = live && c != u && !maybe_nb && d2 > 0.f;
          sx += good ? clip4(g * dx) : 0.f;
          sy += good ? clip4(g * dy) : 0.f;
          if (live && !good) redo |= 1u << q;
        }
        sx *= lr;
        sy *= lr;
        dux += sx;
        duy += sy;
        xu.x += sx;
        xu.y += sy;
        if (!__any_sync(FULL, redo != 0u)) continue;
#pragma unroll
        for (int q = 0; q < SGD_NEG_BLOCK; q++) {
          const int ln = (int)((d0 + (unsigned)(q0 + q) * stride) & 31u);
          int c = __shfl_sync(FULL, pool_c, ln);
          float2 xcq;
          xcq.x = __shfl_sync(FULL, pool_xy.x, ln);
          xcq.y = __shfl_sync(FULL, pool_xy.y, ln);
          if (!((redo >> q) & 1u)) continue;
          unsigned draw = draw32(vbase, q0 + q, 0);
          if (c == u || (c >= rlo && c <= rhi && is_neighbor(nip, nix, u, c))) {
            c = -1;
            for (int t = 1; t < 8; t++) {  // retries 2..8 of this slot
              const unsigned rr = draw32(vbase, q0 + q, t);
              const int cc = (int)__umulhi(rr, (unsigned)n);
              if (cc == u || (cc >= rlo && cc <= rhi && is_neighbor(nip, nix, u, cc))) continue;
              c = cc;
              draw = rr;
              break;
            }
            if (c < 0) continue;
            xcq = xy[c];
          }
          const float dx = xu.x - xcq.x, dy = xu.y - xcq.y;
          const float d2 = dx * dx + dy * dy;
          float gx, gy;
          if (d2 > 0.f) {
            const float g = __fdividef(2.0f * b, (0.001f + d2) * (a * __powf(d2, b) + 1.0f));
            gx = clip4(g * dx);
            gy = clip4(g * dy);
          } else {
            const float th = (float)theta_draw(draw) * (6.283185307179586f / 4294967296.0f);
            float sn, cs;
            __sincosf(th, &sn, &cs);
            gx = 4.0f * cs;
            gy = 4.0f * sn;
          }
          gx *= lr;
          gy *= lr;
          dux += gx;
          duy += gy;
          xu.x += gx;
          xu.y += gy;
        }
      }
    } else
#endif
    for (int q0 = 0; q0 < n_neg; q0 += SGD_NEG_BLOCK) {
      const int nq = min(SGD_NEG_BLOCK, n_neg - q0);
      int cand[SGD_NEG_BLOCK];
      unsigned draw_q[SGD_NEG_BLOCK];
      float2 xc[SGD_NEG_BLOCK];
      unsigned mm = 0;  // slots whose filter bit is set
      if (POOL) {
        // first tries from the warp's pool: slot q reads the vertex and the
        // coordinates of lane (start + (q0 + q) * stride) & 31, stride odd
        // (distinct lanes for up to 32 slots), start / stride from the visit's
        // own draw
        const unsigned d0 = draw32(vbase, 0, 0);
        const unsigned stride = ((d0 >> 5) & 15u) * 2u + 1u;
#pragma unroll
        for (int q = 0; q < SGD_NEG_BLOCK; q++) {
          const int ln = (int)((d0 + (unsigned)(q0 + q) * stride) & 31u);
          cand[q] = __shfl_sync(FULL, pool_c, ln);
          xc[q].x = __shfl_sync(FULL, pool_xy.x, ln);
          xc[q].y = __shfl_sync(FULL, pool_xy.y, ln);
          draw_q[q] = 0;  // (the slow path redraws)
          if (act && q < nq && cand[q] >= rlo && cand[q] <= rhi && filt_maybe<F>(fw, cand[q]))
            mm |= 1u << q;
        }
      } else {
#pragma unroll
        for (int q = 0; q < SGD_NEG_BLOCK; q++) {
          draw_q[q] = draw32(vbase, q0 + q, 0);
          cand[q] = (int)__umulhi(draw_q[q], (unsigned)n);
          if (MODE != REC_HASH && act && q < nq && cand[q] >= rlo && cand[q] <= rhi &&
              filt_maybe<F>(fw, cand[q]))
            mm |= 1u << q;
        }
#pragma unroll
        for (int q = 0; q < SGD_NEG_BLOCK; q++)
          xc[q] = (act && q < nq) ? SGD_LD(&xy[cand[q]]) : make_float2(0.f, 0.f);
      }
      unsigned hset_hit = 0;
      if (MODE == REC_HASH && act) {
        // exact set test: all first probes in flight together, then the
        // (rare) longer chains one by one
        const int4* __restrict__ tab = reinterpret_cast<const int4*>(filt);
        const unsigned hoff = (unsigned)rec.w >> 4, lg = (unsigned)rec.w & 15u;
        const unsigned b0 = hoff >> 2, bmask = (1u << (lg - 2)) - 1u;
        unsigned hb[SGD_NEG_BLOCK];
        int4 x0[SGD_NEG_BLOCK];
#pragma unroll
        for (int q = 0; q < SGD_NEG_BLOCK; q++) {
          hb[q] = hset_bucket(cand[q], lg);
          x0[q] = q < nq ? __ldg(tab + b0 + hb[q]) : make_int4(-1, -1, -1, -1);
        }
#pragma unroll
        for (int q = 0; q < SGD_NEG_BLOCK; q++) {
          int4 x = x0[q];
          unsigned h = hb[q];
          const int c = cand[q];
          // a full bucket of other ids sends the probe to the next bucket
          while (x.x != c && x.y != c && x.z != c && x.w != c && (x.x | x.y | x.z | x.w) >= 0) {
            h = (h + 1) & bmask;
            x = __ldg(tab + b0 + h);
          }
          if (x.x == c || x.y == c || x.z == c || x.w == c) hset_hit |= 1u << q;
        }
      }
      // warp-cooperative neighbour test of the filter hits
      const int cnt = __popc(mm);
      int incl = cnt, total = 0;
      if (MODE != REC_HASH) {  // exact sets need no row search
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(FULL, incl, o);
          if (lane >= o) incl += y;
        }
        total = __shfl_sync(FULL, incl, 31);
      }
      unsigned hit = 0;
      if (total > 0) {  // warp-uniform
        int pos = incl - cnt;
#pragma unroll
        for (int q = 0; q < SGD_NEG_BLOCK; q++)
          if ((mm >> q) & 1u) sh_pairs[wib][pos++] = make_int4(cand[q], rb, re, lane * 8 + q);
        sh_hit[wib][lane] = 0;
        __syncwarp();
        for (int t = lane; t < total; t += 32) {
          const int4 pr = sh_pairs[wib][t];
          int lo = pr.y, len = pr.z - pr.y;
          // binary steps only above SCAN entries (long rows); the rest of the
          // row is read with independent loads: one memory round trip
          // instead of a chain of dependent probes
          while (len > SGD_SCAN) {
            const int half = len >> 1;
            if (__ldg(nix + lo + half) < pr.x) {
              lo += half + 1;
              len -= half + 1;
            } else {
              len = half;
            }
          }
          int x[SGD_SCAN];
#pragma unroll
          for (int q = 0; q < SGD_SCAN; q++) x[q] = q < len ? __ldg(nix + lo + q) : -1;
          bool found = false;
#pragma unroll
          for (int q = 0; q < SGD_SCAN; q++) found |= x[q] == pr.x;
          if (found) atomicOr(&sh_hit[wib][pr.w >> 3], 1u << (pr.w & 7));
        }
        __syncwarp();
        hit = sh_hit[wib][lane];
        __syncwarp();  // the buffers are reused by the next slot block
      }
      if (MODE == REC_HASH) hit = hset_hit;
      if (!act) continue;
#if SGD_LOCKSTEP
      // the block's repulsions all read x_u as it stands after the attraction
      // and the earlier blocks (branch-free: the five gradient chains
      // interleave); a rejected first try or a coincident point takes the
      // sequential path below
      unsigned redo = 0;
      {
        float sx = 0.f, sy = 0.f;
#pragma unroll
        for (int q = 0; q < SGD_NEG_BLOCK; q++) {
          const bool ok = q < nq && cand[q] != u && !((hit >> q) & 1u);
          const float dx = xu.x - xc[q].x, dy = xu.y - xc[q].y;
          const float d2 = dx * dx + dy * dy;
          const float g = __fdividef(2.0f * b, (0.001f + d2) * (a * __powf(d2, b) + 1.0f));
          const bool good = ok && d2 > 0.f;
          sx += good ? clip4(g * dx) : 0.f;
          sy += good ? clip4(g * dy) : 0.f;
          if (q < nq && !good) redo |= 1u << q;
        }
        sx *= lr;
        sy *= lr;
        dux += sx;
        duy += sy;
        xu.x += sx;
        xu.y += sy;
      }
      if (redo == 0) continue;
#else
      const unsigned redo = 0xffffffffu;
#endif
#pragma unroll
      for (int q = 0; q < SGD_NEG_BLOCK; q++) {
        if (q >= nq) break;
        if (!((redo >> q) & 1u)) continue;
        const bool ok = cand[q] != u && !((hit >> q) & 1u);
        int c = ok ? cand[q] : -1;
        // the accepted try's draw (angle source)
        unsigned draw = POOL ? draw32(vbase, q0 + q, 0) : draw_q[q];
        if (!ok) {
          // retries 2..8 of this slot (rare)
          for (int t = 1; t < 8; t++) {
            const unsigned rr = draw32(vbase, q0 + q, t);
            const int cc = (int)__umulhi(rr, (unsigned)n);
            bool nb;
            if (MODE == REC_HASH) {
              const int4* __restrict__ tab = reinterpret_cast<const int4*>(filt);
              const unsigned hoff = (unsigned)rec.w >> 4, lg = (unsigned)rec.w & 15u;
              const unsigned b0 = hoff >> 2;
              unsigned h = hset_bucket(cc, lg);
              int4 x = __ldg(tab + b0 + h);
              while (x.x != cc && x.y != cc && x.z != cc && x.w != cc && (x.x | x.y | x.z | x.w) >= 0) {
                h = (h + 1) & ((1u << (lg - 2)) - 1u);
                x = __ldg(tab + b0 + h);
              }
              nb = x.x == cc || x.y == cc || x.z == cc || x.w == cc;
            } else {
              nb = is_neighbor(nip, nix, u, cc);
            }
            if (cc == u || nb) continue;
            c = cc;
            draw = rr;
            break;
          }
          if (c < 0) continue;
          xc[q] = xy[c];
        }
        const float dx = xu.x - xc[q].x, dy = xu.y - xc[q].y;
        const float d2 = dx * dx + dy * dy;
        float gx, gy;
        if (d2 > 0.f) {
          const float g = __fdividef(2.0f * b, (0.001f + d2) * (a * __powf(d2, b) + 1.0f));
          gx = clip4(g * dx);
          gy = clip4(g * dy);
        } else {
          const float th = (float)theta_draw(draw) * (6.283185307179586f / 4294967296.0f);
          float sn, cs;
          __sincosf(th, &sn, &cs);
          gx = 4.0f * cs;
          gy = 4.0f * sn;
        }
        gx *= lr;
        gy *= lr;
        dux += gx;
        duy += gy;
        xu.x += gx;
        xu.y += gy;
      }
    }
    if (act) {
      if (dux != 0.f || duy != 0.f) push(u, dux, duy);
      if (!isfinite(xu.x) || !isfinite(xu.y)) bad = true;
    }
  }
  if (bad) atomicMin(diverged, epoch);
}

// Small concurrency caps with exact neighbour sets (REC_HASH): ONE VISIT ON
// FOUR LANES.  With n / 4 visits in flight (c1: 625, c3: 25,000) an epoch is
// bound by the length of one visit's dependent chain, not by throughput, so
// the visit's six gradients are spread over a quad: sub-lane 1 takes the
// attraction and slot 1, sub-lanes 0 / 2 / 3 take slots {0, 4} / 2 / 3 (slot
// q on sub-lane q & 3).  Every part reads x_u as the visit found it; a
// sub-lane applies its own slots in order; the quad's deltas are summed by
// two shuffles and pushed once.  Same draws as sgd_epoch_kernel (draw32 of
// the visit base), same rejection rule, same update formulas -- only the
// order inside a visit is relaxed (check (c): tests/test_gpu_parity.py
// quality tests, profiles/r02_ab_sgd_split.log).  8 visits per warp.
__global__ void __launch_bounds__(256, 3)
    sgd_epoch_split_kernel(int n, long long E, float2* __restrict__ xy,
                           const int4* __restrict__ edges, const int4* __restrict__ tab, float a,
                           float b, float lr, int epoch, int n_neg, long long items,
                           long long start, int windowed, unsigned long long seed,
                           int* __restrict__ diverged) {
  constexpr int lanes = 8;
  const long long ntiles = (E + TILE - 1) / TILE;
  Feistel tperm((unsigned long long)ntiles, mix64(seed ^ (0x51ED27ull + (unsigned long long)epoch)));
  const unsigned long long rkey = mix64(seed ^ (0xA5A5A5A5ull * (unsigned long long)(epoch + 1)));
  const int lane = threadIdx.x & 31, vi = lane >> 2, sub = lane & 3;
  bool bad = false;
  const long long gwarp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long stride = (((long long)gridDim.x * blockDim.x) >> 5) * lanes;
  unsigned tile_batch = 0;
  int step = 0;
  for (long long i0 = gwarp * lanes; i0 < items; i0 += stride, step = (step + 1) & 31) {
    const long long i = i0 + vi;
    bool act = i < items;
    long long p = 0;
    if (windowed) {
      p = start + i;
      if (p >= E) p -= E;
    } else {
      if (step == 0) {
        const long long il = i0 + (long long)lane * stride;
        tile_batch = il < items ? (unsigned)tperm((unsigned long long)(il / TILE)) : 0u;
      }
      const long long tile = (long long)__shfl_sync(FULL, tile_batch, step);
      p = tile * TILE + (i - (i0 / TILE) * TILE);
      if (p >= E) act = false;  // partial last tile maps onto itself
    }
    if (!act) p = 0;
    const int4 rec = act ? __ldcs(edges + p) : make_int4(0, 0, 0, 0);
    const int u = rec.x, v = rec.y;
    const float2 x0 = SGD_LD(&xy[u]);
    float2 xu = x0;
    float dux = 0.f, duy = 0.f;
    const unsigned long long vbase = mix64(rkey ^ (unsigned long long)p);
    if (act) {
      const unsigned hoff = (unsigned)rec.w >> 4, lg = (unsigned)rec.w & 15u;
      const unsigned b0 = hoff >> 2, bmask = (1u << (lg - 2)) - 1u;
      // first tries of this sub-lane's slots: bucket and coordinates in flight together
      const int q1 = sub, q2 = sub + 4;
      const unsigned r1 = draw32(vbase, q1, 0), r2 = draw32(vbase, q2, 0);
      const int c1 = (int)__umulhi(r1, (unsigned)n), c2 = (int)__umulhi(r2, (unsigned)n);
      const bool has1 = q1 < n_neg, has2 = q2 < n_neg;
      int4 k1 = make_int4(-1, -1, -1, -1), k2 = k1;
      float2 y1 = make_float2(0.f, 0.f), y2 = y1;
      if (has1) {
        k1 = __ldg(tab + b0 + hset_bucket(c1, lg));
        y1 = SGD_LD(&xy[c1]);
      }
      if (has2) {
        k2 = __ldg(tab + b0 + hset_bucket(c2, lg));
        y2 = SGD_LD(&xy[c2]);
      }
      if (sub == 1) {  // attraction
        const float2 xv = SGD_LD(&xy[v]);
        const float h = __int_as_float(rec.z);
        const float dx = x0.x - xv.x, dy = x0.y - xv.y;
        const float d2 = dx * dx + dy * dy;
        if (d2 > 0.f) {
          const float pb = __powf(d2, b);
          const float g = __fdividef(-2.0f * a * b * h * pb, d2 * (a * pb + 1.0f));
          const float gx = clip4(g * dx) * lr, gy = clip4(g * dy) * lr;
          dux += gx;
          duy += gy;
          atomicAdd(&xy[v], make_float2(-gx, -gy));
          if (!isfinite(xv.x - gx) || !isfinite(xv.y - gy)) bad = true;
        }
      }
      // is c in the head's exact neighbour set?  (first bucket already loaded)
      auto in_set = [&](int c, int4 x) -> bool {
        unsigned hb = hset_bucket(c, lg);
        while (x.x != c && x.y != c && x.z != c && x.w != c && (x.x | x.y | x.z | x.w) >= 0) {
          hb = (hb + 1) & bmask;
          x = __ldg(tab + b0 + hb);
        }
        return x.x == c || x.y == c || x.z == c || x.w == c;
      };
      auto repel = [&](int q, int c, unsigned draw, int4 k, float2 y) {
        if (c == u || in_set(c, k)) {  // retries 2..8 of this slot (rare)
          c = -1;
          for (int t = 1; t < 8; t++) {
            const unsigned rr = draw32(vbase, q, t);
            const int cc = (int)__umulhi(rr, (unsigned)n);
            if (cc == u || in_set(cc, __ldg(tab + b0 + hset_bucket(cc, lg)))) continue;
            c = cc;
            draw = rr;
            break;
          }
          if (c < 0) return;
          y = xy[c];
        }
        const float dx = xu.x - y.x, dy = xu.y - y.y;
        const float d2 = dx * dx + dy * dy;
        float gx, gy;
        if (d2 > 0.f) {
          const float g = __fdividef(2.0f * b, (0.001f + d2) * (a * __powf(d2, b) + 1.0f));
          gx = clip4(g * dx);
          gy = clip4(g * dy);
        } else {
          const float th = (float)theta_draw(draw) * (6.283185307179586f / 4294967296.0f);
          float sn, cs;
          __sincosf(th, &sn, &cs);
          gx = 4.0f * cs;
          gy = 4.0f * sn;
        }
        gx *= lr;
        gy *= lr;
        dux += gx;
        duy += gy;
        xu.x += gx;
        xu.y += gy;
      };
      if (has1) repel(q1, c1, r1, k1, y1);
      if (has2) repel(q2, c2, r2, k2, y2);
      for (int q = sub + 8; q < n_neg; q += 4) {  // more than 8 negatives
        const unsigned rr = draw32(vbase, q, 0);
        const int cc = (int)__umulhi(rr, (unsigned)n);
        repel(q, cc, rr, __ldg(tab + b0 + hset_bucket(cc, lg)), SGD_LD(&xy[cc]));
      }
    }
    // the quad's deltas, summed on every lane (lanes of inactive visits add zeros)
    dux += __shfl_xor_sync(FULL, dux, 1);
    duy += __shfl_xor_sync(FULL, duy, 1);
    dux += __shfl_xor_sync(FULL, dux, 2);
    duy += __shfl_xor_sync(FULL, duy, 2);
    if (act && sub == 0) {
      if (dux != 0.f || duy != 0.f) atomicAdd(&xy[u], make_float2(dux, duy));
      if (!isfinite(x0.x + dux) || !isfinite(x0.y + duy)) bad = true;
    }
  }
  if (bad) atomicMin(diverged, epoch);
}

// deterministic mode: x += acc * 2^-32, acc = 0, finiteness check
__global__ void det_apply_kernel(int n, float2* __restrict__ xy, long long* __restrict__ acc,
                                 int epoch, int* __restrict__ diverged) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const long long ax = acc[2 * (long long)v], ay = acc[2 * (long long)v + 1];
    if (ax == 0 && ay == 0) continue;
    float2 x = xy[v];
    x.x += (float)((double)ax * 2.3283064365386963e-10);
    x.y += (float)((double)ay * 2.3283064365386963e-10);
    xy[v] = x;
    acc[2 * (long long)v] = 0;
    acc[2 * (long long)v + 1] = 0;
    if (!isfinite(x.x) || !isfinite(x.y)) atomicMin(diverged, epoch);
  }
}

__global__ void visit_order_kernel(long long E, int epoch, long long items, long long start,
                                   int windowed, unsigned long long seed,
                                   long long* __restrict__ out) {
  const long long ntiles = (E + TILE - 1) / TILE;
  Feistel tperm((unsigned long long)ntiles, mix64(seed ^ (0x51ED27ull + (unsigned long long)epoch)));
  // full mode: compact the tile order (the partial last tile keeps its slot)
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < items;
       i += (long long)gridDim.x * blockDim.x) {
    long long p;
    if (windowed) {
      p = start + i;
      if (p >= E) p -= E;
      out[i] = p;
    } else {
      const long long t = i / TILE;
      p = (long long)tperm((unsigned long long)t) * TILE + (i - t * TILE);
      out[i] = p < E ? p : -1;
    }
  }
}

unsigned grid_for(long long items, long long max_threads = 0) {
  long long b = (items + 255) / 256;
  if (b > 148LL * 8) b = 148LL * 8;
  if (max_threads > 0 && b * 256 > max_threads) b = (max_threads + 255) / 256;
  if (b < 1) b = 1;
  return (unsigned)b;
}

unsigned block_for(long long max_threads) {
  if (max_threads > 0 && max_threads < 256) return (unsigned)(((max_threads + 31) / 32) * 32);
  return 256;
}

}  // namespace
}  // namespace gu

using namespace gu;

// visits per warp of an epoch launch: a cap below the resident-thread
// capacity (4 blocks of 256 per SM at 64 registers) runs 16 visits per warp
// on cap * 2 threads -- the same visits in flight, more warps to hide
// latency (measured best on c3; 8 lanes slows full epochs).
// GU_SGD_MIN_LANES=32 turns it off.
static int sgd_lanes(long long concurrency) {
  const long long resident = 148LL * SGD_MIN_BLOCKS * 256;
  static const int min_lanes = [] {
    const char* v = getenv("GU_SGD_MIN_LANES");
    return (v && atoi(v) >= 32) ? 32 : 16;
  }();
  // 8 visits per warp when the cap fits the 3-CTA/SM kernel: the same visits
  // in flight as 4x the warps of the 32-lane kernel (c3 SL 200 epochs 8.1 ->
  // 7.8 ms, c1 GUMAP 15.1 -> 14.7 ms: profiles/r02_ab_sgd_lanes8.log)
  if (concurrency > 0 && concurrency < resident && min_lanes == 16 &&
      (concurrency * 32) / 8 <= 148LL * 3 * 256)
    return 8;
  if (concurrency > 0 && concurrency < resident && min_lanes == 16 &&
      (concurrency * 32) / 16 <= 148LL * 2 * 256)  // fits the 2-CTA/SM kernel
    return 16;
  return 32;
}

extern "C" int32_t gu_sgd_record_bytes_for(int64_t concurrency) {
  // GPU-filling epochs stream 32-byte records with the in-record filter;
  // small caps keep 16-byte records and the gathered 64-bit table
  return sgd_lanes(concurrency) == 32 ? 32 : 16;
}

extern "C" int gu_sgd_prepare_edges(int64_t E, const int32_t* sym_src, const int32_t* sym_dst,
                                    const double* sym_w, const int32_t* nbr_indptr,
                                    const int32_t* nbr_indices, const int32_t* relabel,
                                    int32_t record_mode, uint64_t seed, void* edges,
                                    int32_t* perm_out, void* stream) {
  if (E < 0 || E >= INT_MAX || record_mode < REC_TABLE || record_mode > REC_RANGE) {
    set_error("gu_sgd_prepare_edges: unsupported E=%lld / record_mode=%d", (long long)E,
              record_mode);
    return GU_ERR_UNSUPPORTED;
  }
  if (E == 0) return GU_OK;
  prepare_edges_kernel<<<grid_for(E), 256, 0, (cudaStream_t)stream>>>(
      E, sym_src, sym_dst, sym_w, nbr_indptr, nbr_indices, relabel, record_mode,
      mix64(seed ^ 0xED6E5ull), (int4*)edges, perm_out);
  GU_CHECK_LAUNCH("prepare_edges_kernel");
  return GU_OK;
}

extern "C" int gu_sgd_prepare_edges_local(int64_t n, int64_t E, const double* sym_w,
                                          const int32_t* new_indptr, const int32_t* new_indices,
                                          const int32_t* order, const int32_t* nbr_indptr,
                                          const int32_t* nbr_indices, int64_t block,
                                          uint64_t seed, void* edges, int32_t* perm_out,
                                          void* stream) {
  if (n < 1 || n >= INT_MAX || E < 0 || E >= INT_MAX || block < 1) {
    set_error("gu_sgd_prepare_edges_local: bad arguments");
    return GU_ERR_ARG;
  }
  if (E == 0) return GU_OK;
  prepare_edges_local<<<grid_for(E), 256, 0, (cudaStream_t)stream>>>(
      E, sym_w, (int)n, new_indptr, new_indices, order, nbr_indptr, nbr_indices, block,
      mix64(seed ^ 0xED6E5ull), (int4*)edges, perm_out);
  GU_CHECK_LAUNCH("prepare_edges_local");
  return GU_OK;
}

static void epoch_range(int64_t E, int32_t epoch, int64_t window, int32_t windowed,
                        long long* items, long long* start) {
  if (windowed) {
    *items = window;
    // j advances by window each epoch, modulo E (layout.py:336-337)
    *start = (long long)(((__int128)epoch * (__int128)window) % (__int128)E);
  } else {
    *items = ((E + TILE - 1) / TILE) * TILE;
    *start = 0;
  }
}

namespace gu {
namespace {
__global__ void hset_sizes(int n, const int* __restrict__ nip, int* __restrict__ sz,
                           int* __restrict__ bad) {
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const int d = nip[v + 1] - nip[v];
    int S = 0;
    if (d > 0) {
      S = 4;
      while (S < 4 * d && S < (1 << 16)) S <<= 1;
      if (S < 4 * d || S > (1 << 15)) atomicExch(bad, 1);  // log2 S must fit 4 bits
    }
    sz[v] = S;
  }
}
// one warp per vertex: its neighbour ids inserted by CAS with linear probing
__global__ void hset_build(int n, const int* __restrict__ nip, const int* __restrict__ nix,
                           const int* __restrict__ off, int* __restrict__ tab) {
  const int lane = threadIdx.x & 31;
  for (long long v = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n;
       v += ((long long)gridDim.x * blockDim.x) >> 5) {
    const int b = nip[v], e = nip[v + 1];
    const int S = off[v + 1] - off[v];
    if (S == 0) continue;
    const unsigned lg = 31u - (unsigned)__clz(S), bmask = ((unsigned)S >> 2) - 1u;
    int* const t = tab + off[v];
    for (int p = b + lane; p < e; p += 32) {
      const int c = nix[p];
      unsigned h = hset_bucket(c, lg);
      for (bool done = false; !done; h = (h + 1) & bmask) {
        for (int j = 0; j < 4 && !done; j++) {
          const int old = atomicCAS(t + 4 * h + j, -1, c);
          done = old == -1 || old == c;
        }
      }
    }
  }
}
__global__ void prepare_edges_hash_kernel(long long E, const int* __restrict__ src,
                                          const int* __restrict__ dst,
                                          const double* __restrict__ w,
                                          const int* __restrict__ off, unsigned long long key,
                                          int4* __restrict__ out, int* __restrict__ perm_out) {
  Feistel perm((unsigned long long)E, key);
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < E;
       p += (long long)gridDim.x * blockDim.x) {
    const long long e = (long long)perm((unsigned long long)p);
    const int u = src[e], v = dst[e];
    const int o = off[u], S = off[u + 1] - o;
    const int lg = S > 0 ? 31 - __clz(S) : 0;
    out[p] = make_int4(u, v, __float_as_int((float)w[e]), (o << 4) | lg);
    if (perm_out) perm_out[p] = (int)e;
  }
}
}  // namespace
}  // namespace gu

extern "C" int gu_sgd_neighbor_hash_layout(int64_t n, const int32_t* nbr_indptr, int32_t* off,
                                           int64_t* host_slots, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n <= 0 || n >= INT_MAX) {
    set_error("gu_sgd_neighbor_hash_layout: bad n=%lld", (long long)n);
    return GU_ERR_ARG;
  }
  int* bad = nullptr;  // [0] flag, [1 ..] the sizes (scanned into off)
  void* tmp = nullptr;
  size_t tb = 0;
  GU_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, tb, off, off, (int)n + 1, st));
  GU_CHECK(cudaMallocAsync((void**)&bad, sizeof(int) * (size_t)(n + 2), st));
  GU_CHECK(cudaMallocAsync(&tmp, tb, st));
  int* sz = bad + 1;
  GU_CHECK(cudaMemsetAsync(bad, 0, sizeof(int) * (size_t)(n + 2), st));
  hset_sizes<<<grid_for(n), 256, 0, st>>>((int)n, nbr_indptr, sz, bad);
  GU_CHECK_LAUNCH("hset_sizes");
  // total slots = 4 deg rounded up <= 8 * nnz: fits int32 whenever nnz < 2^28
  GU_CHECK(cub::DeviceScan::ExclusiveSum(tmp, tb, sz, off, (int)n + 1, st));
  int h_bad = 0, h_tot = 0;
  GU_CHECK(cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  GU_CHECK(cudaMemcpyAsync(&h_tot, off + n, sizeof(int), cudaMemcpyDeviceToHost, st));
  GU_CHECK(cudaFreeAsync(bad, st));
  GU_CHECK(cudaFreeAsync(tmp, st));
  GU_CHECK(cudaStreamSynchronize(st));
  if (h_bad || h_tot < 0 || h_tot >= (1 << 28)) {
    set_error("gu_sgd_neighbor_hash_layout: a row above 8192 ids or 2^28 slots in total");
    return GU_ERR_UNSUPPORTED;
  }
  *host_slots = h_tot;
  return GU_OK;
}

extern "C" int gu_sgd_neighbor_hash(int64_t n, const int32_t* nbr_indptr,
                                    const int32_t* nbr_indices, const int32_t* off,
                                    int32_t* table, int64_t slots, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n <= 0 || n >= INT_MAX || slots < 0) {
    set_error("gu_sgd_neighbor_hash: bad arguments");
    return GU_ERR_ARG;
  }
  GU_CHECK(cudaMemsetAsync(table, 0xff, sizeof(int32_t) * (size_t)slots, st));
  hset_build<<<grid_for(n * 32), 256, 0, st>>>((int)n, nbr_indptr, nbr_indices, off, table);
  GU_CHECK_LAUNCH("hset_build");
  return GU_OK;
}

extern "C" int gu_sgd_prepare_edges_hash(int64_t E, const int32_t* sym_src,
                                         const int32_t* sym_dst, const double* sym_w,
                                         const int32_t* off, uint64_t seed, void* edges,
                                         int32_t* perm_out, void* stream) {
  if (E < 0 || E >= INT_MAX) {
    set_error("gu_sgd_prepare_edges_hash: unsupported E=%lld", (long long)E);
    return GU_ERR_UNSUPPORTED;
  }
  if (E == 0) return GU_OK;
  prepare_edges_hash_kernel<<<grid_for(E), 256, 0, (cudaStream_t)stream>>>(
      E, sym_src, sym_dst, sym_w, off, seed, (int4*)edges, perm_out);
  GU_CHECK_LAUNCH("prepare_edges_hash_kernel");
  return GU_OK;
}

extern "C" int gu_sgd_neighbor_filter(int64_t n, const int32_t* nbr_indptr,
                                      const int32_t* nbr_indices, void* filter_out, void* stream) {
  if (n <= 0 || n >= INT_MAX) {
    set_error("gu_sgd_neighbor_filter: bad n");
    return GU_ERR_ARG;
  }
  neighbor_filter_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(
      (int)n, nbr_indptr, nbr_indices, (FiltWord*)filter_out);
  GU_CHECK_LAUNCH("neighbor_filter_kernel");
  return GU_OK;
}

typedef void (*EpochKernel)(int, long long, float2*, const int4*, const int*, const int*,
                            const FiltWord*, float, float, float, int, int, long long, long long,
                            int, unsigned long long, int*, long long, long long*);

static EpochKernel epoch_kernel(int lanes, int mode) {
  if (lanes == 32)
    return mode == REC_RANGE   ? sgd_epoch_kernel<32, SGD_MIN_BLOCKS, REC_RANGE>
           : mode == REC_BLOOM ? sgd_epoch_kernel<32, SGD_MIN_BLOCKS, REC_BLOOM>
           : mode == REC_HASH  ? sgd_epoch_kernel<32, SGD_MIN_BLOCKS, REC_HASH>
                               : sgd_epoch_kernel<32, SGD_MIN_BLOCKS, REC_TABLE>;
  if (lanes == 8)
    return mode == REC_RANGE   ? sgd_epoch_kernel<8, 3, REC_RANGE>
           : mode == REC_BLOOM ? sgd_epoch_kernel<8, 3, REC_BLOOM>
           : mode == REC_HASH  ? sgd_epoch_kernel<8, 3, REC_HASH>
                               : sgd_epoch_kernel<8, 3, REC_TABLE>;
  return mode == REC_RANGE   ? sgd_epoch_kernel<16, 2, REC_RANGE>
         : mode == REC_BLOOM ? sgd_epoch_kernel<16, 2, REC_BLOOM>
         : mode == REC_HASH  ? sgd_epoch_kernel<16, 2, REC_HASH>
                             : sgd_epoch_kernel<16, 2, REC_TABLE>;
}

extern "C" int gu_sgd_epochs(int64_t n, int64_t E, float* coords_xy, const void* edges,
                             int32_t record_mode, const int32_t* nbr_indptr,
                             const int32_t* nbr_indices, const void* nbr_filter, float a,
                             float b, float lr0, int32_t t, int32_t epoch_begin, int32_t epoch_end,
                             int32_t n_neg, int64_t window, int32_t windowed, uint64_t seed,
                             int64_t concurrency, int32_t* diverged, void* stream) {
  if (n <= 0 || n >= INT_MAX || E < 0 || t < 0 || epoch_begin < 0 || epoch_end > t ||
      record_mode < REC_TABLE || record_mode > REC_HASH || (windowed && (window < 1 || window > E))) {
    set_error("gu_sgd_epochs: bad arguments");
    return GU_ERR_ARG;
  }
  if (E == 0) return GU_OK;
  cudaStream_t st = (cudaStream_t)stream;
  for (int e = epoch_begin; e < epoch_end; e++) {
    // lr = learning_rate * (1 - it / t), layout.py:334 (float64 on host)
    const float lr = (float)((double)lr0 * (1.0 - (double)e / (double)t));
    long long items, start;
    epoch_range(E, e, window, windowed, &items, &start);
    const int lanes = sgd_lanes(concurrency);
    const long long threads = concurrency > 0 ? (concurrency * 32 + lanes - 1) / lanes : 0;
    const unsigned bs = block_for(threads);
    const unsigned gs = bs < 256 ? 1u : grid_for((items * 32 + lanes - 1) / lanes, threads);
    // small caps on exact neighbour sets: one visit on four lanes
    // (GU_SGD_SPLIT=0: the one-lane-per-visit kernel, for comparison)
    static const bool split = [] {
      const char* v = getenv("GU_SGD_SPLIT");
      return !(v && v[0] == '0');
    }();
    if (split && lanes == 8 && record_mode == REC_HASH && bs == 256) {
      sgd_epoch_split_kernel<<<gs, bs, 0, st>>>((int)n, E, (float2*)coords_xy, (const int4*)edges,
                                                (const int4*)nbr_filter, a, b, lr, e, n_neg, items,
                                                start, windowed, seed, diverged);
      GU_CHECK_LAUNCH("sgd_epoch_split_kernel");
      continue;
    }
    EpochKernel kern = epoch_kernel(lanes, record_mode);
    kern<<<gs, bs, 0, st>>>((int)n, E, (float2*)coords_xy, (const int4*)edges, nbr_indptr,
                            nbr_indices, (const FiltWord*)nbr_filter, a, b, lr, e, n_neg, items,
                            start, windowed, seed, diverged, 0LL, nullptr);
    GU_CHECK_LAUNCH("sgd_epoch_kernel");
  }
  return GU_OK;
}

extern "C" int gu_sgd_epochs_deterministic(int64_t n, int64_t E, float* coords_xy,
                                           const void* edges, int32_t record_mode,
                                           const int32_t* nbr_indptr,
                                           const int32_t* nbr_indices, const void* nbr_filter,
                                           float a, float b, float lr0, int32_t t,
                                           int32_t epoch_begin, int32_t epoch_end, int32_t n_neg,
                                           int64_t window, int32_t windowed, uint64_t seed,
                                           int64_t batch, int64_t* acc, int32_t* diverged,
                                           void* stream) {
  if (n <= 0 || n >= INT_MAX || E < 0 || t < 0 || epoch_begin < 0 || epoch_end > t ||
      batch < 32 || !acc || record_mode < REC_TABLE || record_mode > REC_HASH ||
      (windowed && (window < 1 || window > E))) {
    set_error("gu_sgd_epochs_deterministic: bad arguments");
    return GU_ERR_ARG;
  }
  if (E == 0) return GU_OK;
  cudaStream_t st = (cudaStream_t)stream;
  batch = (batch / 32) * 32;  // warp steps never straddle a tile boundary
  for (int e = epoch_begin; e < epoch_end; e++) {
    const float lr = (float)((double)lr0 * (1.0 - (double)e / (double)t));
    long long items, start;
    epoch_range(E, e, window, windowed, &items, &start);
    for (long long b0 = 0; b0 < items; b0 += batch) {
      const long long b1 = b0 + batch < items ? b0 + batch : items;
      const long long threads = b1 - b0;
      const unsigned bs = block_for(threads);
      const unsigned gs = bs < 256 ? 1u : grid_for(threads, threads);
      epoch_kernel(32, record_mode)<<<gs, bs, 0, st>>>(
          (int)n, E, (float2*)coords_xy, (const int4*)edges, nbr_indptr, nbr_indices,
          (const FiltWord*)nbr_filter, a, b, lr, e, n_neg, b1, start, windowed, seed, diverged,
          b0, (long long*)acc);
      GU_CHECK_LAUNCH("sgd_epoch_kernel(deterministic)");
      det_apply_kernel<<<grid_for(n), 256, 0, st>>>((int)n, (float2*)coords_xy,
                                                    (long long*)acc, e, diverged);
      GU_CHECK_LAUNCH("det_apply_kernel");
    }
  }
  return GU_OK;
}

extern "C" int gu_sgd_visit_order(int64_t E, int32_t epoch, int64_t window, int32_t windowed,
                                  uint64_t seed, int64_t* out_order, void* stream) {
  if (E <= 0) return GU_OK;
  long long items, start;
  epoch_range(E, epoch, window, windowed, &items, &start);
  visit_order_kernel<<<grid_for(items), 256, 0, (cudaStream_t)stream>>>(
      E, epoch, items, start, windowed, seed, (long long*)out_order);
  GU_CHECK_LAUNCH("visit_order_kernel");
  return GU_OK;
}
