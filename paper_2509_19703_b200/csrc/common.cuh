// common.cuh -- shared device helpers for libgumap (sm_100a).
//
// RNG restatements (bit-exact with the reference's streams):
//   splitmix64       /root/reference/pkg/src/graph_umap/_kernels.py:13-30
//   numpy SeedSequence + PCG64 + Generator.permutation (numpy 2.3.5), used by
//   knn_from_full_distances (neighbors.py:213-216) for k-th distance ties.
// Counter-based RNG for the Hogwild SGD epochs: sgd.cu draw32 (per-visit 64-bit finaliser, 32-bit per draw).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define GU_INF32 0x7fffffff

namespace gu {

// ------------------------------------------- internal cross-file launchers
// full_bfs.cu: one fused stress pass over every source (metrics.cu)
int stress_bfs_pass(int64_t n, const int32_t* indptr, const int32_t* indices, const double* xy,
                    int pass2, const double* scale, void* acc, int* flag, void* workspace,
                    size_t ws_bytes, int ctas, const int32_t* sources, int64_t nsources,
                    cudaStream_t st);
size_t stress_bfs_workspace(int64_t n, int ctas);

// --------------------------------------------------------------- errors
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* what);
#define GU_CHECK(call)                                  \
  do {                                                  \
    cudaError_t _e = (call);                            \
    if (_e != cudaSuccess) return gu::cuda_status(_e, #call); \
  } while (0)
#define GU_CHECK_LAUNCH(what)                           \
  do {                                                  \
    cudaError_t _e = cudaGetLastError();                \
    if (_e != cudaSuccess) return gu::cuda_status(_e, what); \
  } while (0)

enum Status : int {
  GU_OK = 0,
  GU_ERR_ARG = 1,
  GU_ERR_CUDA = 2,
  GU_ERR_WORKSPACE = 3,
  GU_ERR_UNSUPPORTED = 4,
};

// ------------------------------------------------------------ splitmix64
constexpr unsigned long long SPLIT_GAMMA = 0x9E3779B97F4A7C15ULL;
constexpr unsigned long long SPLIT_MUL1 = 0xBF58476D1CE4E5B9ULL;
constexpr unsigned long long SPLIT_MUL2 = 0x94D049BB133111EBULL;

__host__ __device__ __forceinline__ unsigned long long splitmix_next(unsigned long long& state) {
  state += SPLIT_GAMMA;
  unsigned long long z = state;
  z = (z ^ (z >> 30)) * SPLIT_MUL1;
  z = (z ^ (z >> 27)) * SPLIT_MUL2;
  return z ^ (z >> 31);
}

// --------------------------------------------- numpy SeedSequence / PCG64
struct u128 {
  uint64_t hi, lo;
};
__device__ __forceinline__ u128 mul128(u128 a, u128 b) {
  u128 r;
  r.lo = a.lo * b.lo;
  r.hi = __umul64hi(a.lo, b.lo) + a.hi * b.lo + a.lo * b.hi;
  return r;
}
__device__ __forceinline__ u128 add128(u128 a, u128 b) {
  u128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
  return r;
}

struct Pcg64 {
  u128 state, inc;
  uint32_t buf32;
  bool has32;

  __device__ __forceinline__ void step() {
    const u128 M = {0x2360ED051FC65DA4ULL, 0x4385DF649FCCF645ULL};
    state = add128(mul128(state, M), inc);
  }
  __device__ __forceinline__ uint64_t next64() {
    step();
    uint64_t x = state.hi ^ state.lo;
    unsigned rot = (unsigned)(state.hi >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
  __device__ __forceinline__ uint32_t next32() {
    if (has32) {
      has32 = false;
      return buf32;
    }
    uint64_t v = next64();
    has32 = true;
    buf32 = (uint32_t)(v >> 32);
    return (uint32_t)v;
  }
  // numpy random_interval (distributions.c): masked rejection
  __device__ __forceinline__ uint64_t interval(uint64_t max) {
    if (max == 0) return 0;
    uint64_t mask = max;
    mask |= mask >> 1;
    mask |= mask >> 2;
    mask |= mask >> 4;
    mask |= mask >> 8;
    mask |= mask >> 16;
    mask |= mask >> 32;
    uint64_t v;
    if (max <= 0xffffffffULL) {
      while ((v = (next32() & mask)) > max) {
      }
    } else {
      while ((v = (next64() & mask)) > max) {
      }
    }
    return v;
  }
};

// SeedSequence(entropy=seed, spawn_key=(key,)).generate_state(4, uint64) ->
// PCG64 seeding (pcg64_set_seed: state=0; inc=(seq<<1)|1; step; +=seed; step)
__device__ __forceinline__ uint32_t ss_hashmix(uint32_t v, uint32_t& hc) {
  v ^= hc;
  hc *= 0x931e8875u;
  v *= hc;
  v ^= v >> 16;
  return v;
}
__device__ __forceinline__ uint32_t ss_mix(uint32_t x, uint32_t y) {
  uint32_t r = 0xca01f9ddu * x - 0x4973f715u * y;
  r ^= r >> 16;
  return r;
}
// has_key false: SeedSequence(seed) without a spawn key (np.random.default_rng(seed))
__device__ inline void pcg64_from_seedseq(Pcg64& r, uint64_t seed, uint64_t key,
                                          bool has_key = true) {
  uint32_t ent[8];
  int ne = 0;
  if (seed == 0) {
    ent[ne++] = 0;
  } else {
    uint64_t x = seed;
    while (x) {
      ent[ne++] = (uint32_t)x;
      x >>= 32;
    }
  }
  while (ne < 4) ent[ne++] = 0;  // (without a key: hashmix(0) fills the pool alike)
  if (!has_key) {
  } else if (key == 0) {
    ent[ne++] = 0;
  } else {
    uint64_t x = key;
    while (x) {
      ent[ne++] = (uint32_t)x;
      x >>= 32;
    }
  }
  uint32_t pool[4];
  uint32_t hc = 0x43b0d7e5u;
#pragma unroll
  for (int i = 0; i < 4; i++) pool[i] = ss_hashmix(ent[i], hc);
#pragma unroll
  for (int s = 0; s < 4; s++)
#pragma unroll
    for (int d = 0; d < 4; d++)
      if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], hc));
  for (int s = 4; s < ne; s++)
#pragma unroll
    for (int d = 0; d < 4; d++) pool[d] = ss_mix(pool[d], ss_hashmix(ent[s], hc));
  uint32_t st[8];
  uint32_t hb = 0x8b51f9ddu;
#pragma unroll
  for (int i = 0; i < 8; i++) {
    uint32_t v = pool[i & 3];
    v ^= hb;
    hb *= 0x58f38dedu;
    v *= hb;
    v ^= v >> 16;
    st[i] = v;
  }
  uint64_t w0 = (uint64_t)st[0] | ((uint64_t)st[1] << 32);
  uint64_t w1 = (uint64_t)st[2] | ((uint64_t)st[3] << 32);
  uint64_t w2 = (uint64_t)st[4] | ((uint64_t)st[5] << 32);
  uint64_t w3 = (uint64_t)st[6] | ((uint64_t)st[7] << 32);
  u128 initstate = {w0, w1};
  u128 initseq = {w2, w3};
  r.state = {0, 0};
  r.inc = {(initseq.hi << 1) | (initseq.lo >> 63), (initseq.lo << 1) | 1ull};
  r.step();
  r.state = add128(r.state, initstate);
  r.step();
  r.has32 = false;
  r.buf32 = 0;
}


// PCG64 jump ahead by `delta` steps (LCG power by squaring, mod 2^128)
__device__ inline void pcg64_advance(Pcg64& r, uint64_t delta) {
  const u128 M = {0x2360ED051FC65DA4ULL, 0x4385DF649FCCF645ULL};
  u128 acc_mult = {0, 1}, acc_plus = {0, 0}, cur_mult = M, cur_plus = r.inc;
  while (delta) {
    if (delta & 1ull) {
      acc_mult = mul128(acc_mult, cur_mult);
      acc_plus = add128(mul128(acc_plus, cur_mult), cur_plus);
    }
    cur_plus = mul128(add128(cur_mult, u128{0, 1}), cur_plus);
    cur_mult = mul128(cur_mult, cur_mult);
    delta >>= 1;
  }
  r.state = add128(mul128(acc_mult, r.state), acc_plus);
}

// ------------------------------------------------------------ warp utils
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane_id() >= o) v += t;
  }
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---- memoised-sigma profile table of K5 (smooth.cu), read back by K6
// (symmetrize.cu).  Lives in the caller's gu_smooth_knn workspace, followed
// (256-byte aligned) by one int slot per row (-1: the row was solved directly).
constexpr int SIG_TABLE = 8192;
constexpr unsigned long long SIG_EMPTY = 0ull;
struct SigTable {
  unsigned long long key[SIG_TABLE];
  long long rep[SIG_TABLE];
  double val[SIG_TABLE];
  double rho[SIG_TABLE];
  double w[SIG_TABLE][4];    // weight of each run
  unsigned ends[SIG_TABLE];  // cumulative run ends, 8 bits each (255 past the last run)
};
constexpr size_t SIG_TABLE_BYTES = (sizeof(SigTable) + 255) & ~(size_t)255;

// weight of entry `i` (position inside its row) of a row with profile `slot`:
// the precomputed weight of the run that holds position i
__device__ __forceinline__ double memo_weight(const SigTable* __restrict__ tab, int slot, unsigned i) {
  const unsigned ends = tab->ends[slot];
  const int j = (i >= (ends & 255u)) + (i >= ((ends >> 8) & 255u)) + (i >= ((ends >> 16) & 255u));
  return tab->w[slot][j];
}

}  // namespace gu
