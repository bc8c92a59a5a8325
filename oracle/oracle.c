/*
 * oracle.c -- CPU restatement of the graph_umap hot path (TEST INFRASTRUCTURE).
 *
 * This file is the parity checker, never the product.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference arm
 * may load it.  The product path (paper_2509_19703_b200) never imports, links
 * or executes anything under oracle/.
 *
 * Each function restates one reference routine (paths relative to
 * /root/reference/pkg/src/graph_umap):
 *   or_apsp_rows          _kernels.py:33-57    (queue BFS rows, INF32 sentinel)
 *   or_partial_bfs_all    _kernels.py:60-131   (truncated BFS, splitmix64 partial
 *                                               Fisher-Yates on the crossing level,
 *                                               (dist,id) sort)
 *   or_knn_select_row     neighbors.py:199-221 (k-th distance ties via numpy
 *                                               SeedSequence -> PCG64 -> permutation)
 *   or_full_knn           apsp row + knn_select_row fused per source (no n x n)
 *   or_smooth_rows        neighbors.py:261-311 (rho / sigma bisection, numpy
 *                                               pairwise row sums, libm exp)
 *   or_fuzzy_union        neighbors.py:320-350 (dedupe, h = (a+b) - a*b over both
 *                                               orientations, zeros dropped, (src,dst))
 *   or_sgd_sweep          _kernels.py:158-223  (sequential float64 SGD, logs the
 *                                               accepted negatives and thetas)
 *   or_sgd_replay         same arithmetic, negatives / thetas supplied
 *
 * Third-party arithmetic restated (numpy 2.3.5, the version installed here):
 *   numpy/random/bit_generator.pyx  SeedSequence mix_entropy / generate_state
 *   numpy/random/src/pcg64          PCG64 XSL-RR 128/64, next_uint32 buffering
 *   numpy/random/_generator.pyx     shuffle: for i=n-1..1 j=random_interval(i)
 *   numpy/_core/src/umath/loops_utils.h.src  pairwise_sum (8 accumulators)
 *
 * Build: oracle/Makefile (gcc -O2 -pthread -ffp-contract=off).  FP contraction
 * must stay off: numba compiles the reference without fastmath.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

/* ------------------------------------------------- tiny dynamic parallel-for */
typedef void (*range_fn)(void *ctx, int64_t begin, int64_t end, void *scratch);
typedef struct {
  range_fn fn;
  void *ctx;
  int64_t begin, end, grain;
  int64_t next; /* atomic */
  size_t scratch_bytes;
} pfor_t;

static void *pfor_worker(void *arg) {
  pfor_t *p = (pfor_t *)arg;
  void *scratch = p->scratch_bytes ? calloc(1, p->scratch_bytes) : NULL;
  for (;;) {
    int64_t b = __atomic_fetch_add(&p->next, p->grain, __ATOMIC_RELAXED);
    if (b >= p->end) break;
    int64_t e = b + p->grain < p->end ? b + p->grain : p->end;
    p->fn(p->ctx, b, e, scratch);
  }
  free(scratch);
  return NULL;
}

static void parallel_for(int nthreads, int64_t begin, int64_t end, int64_t grain,
                         size_t scratch_bytes, range_fn fn, void *ctx) {
  pfor_t p = {fn, ctx, begin, end, grain > 0 ? grain : 1, begin, scratch_bytes};
  if (nthreads <= 1 || end - begin <= p.grain) {
    pfor_worker(&p);
    return;
  }
  pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
  for (int i = 0; i < nthreads; i++) pthread_create(&th[i], NULL, pfor_worker, &p);
  for (int i = 0; i < nthreads; i++) pthread_join(th[i], NULL);
  free(th);
}

#define INF32 0x7fffffff

/* ---------------------------------------------------------------- splitmix64 */
static const uint64_t SPLIT_GAMMA = 0x9E3779B97F4A7C15ULL;
static const uint64_t SPLIT_MUL1 = 0xBF58476D1CE4E5B9ULL;
static const uint64_t SPLIT_MUL2 = 0x94D049BB133111EBULL;

/* _kernels.py:18-25 */
static inline uint64_t sm_next(uint64_t *state) {
  *state += SPLIT_GAMMA;
  uint64_t z = *state;
  z = (z ^ (z >> 30)) * SPLIT_MUL1;
  z = (z ^ (z >> 27)) * SPLIT_MUL2;
  return z ^ (z >> 31);
}
/* _kernels.py:28-30 */
static inline double sm_next_float(uint64_t *state) {
  return (double)(sm_next(state) >> 11) * (1.0 / 9007199254740992.0);
}

/* ----------------------------------------------------------- full BFS rows */
/* _kernels.py:33-57: row[s]=0, FIFO queue, unreachable stays INF32. */
static void bfs_row(int64_t n, const int64_t *indptr, const int32_t *indices,
                    int64_t s, int32_t *row, int32_t *queue) {
  for (int64_t i = 0; i < n; i++) row[i] = INF32;
  row[s] = 0;
  queue[0] = (int32_t)s;
  int64_t head = 0, tail = 1;
  while (head < tail) {
    int32_t u = queue[head++];
    int32_t du = row[u] + 1;
    for (int64_t p = indptr[u]; p < indptr[u + 1]; p++) {
      int32_t v = indices[p];
      if (row[v] == INF32) {
        row[v] = du;
        queue[tail++] = v;
      }
    }
  }
}

typedef struct {
  int64_t n;
  const int64_t *indptr;
  const int32_t *indices;
  const int64_t *sources;
  int32_t *out;
} apsp_ctx;
static void apsp_range(void *c, int64_t b, int64_t e, void *scratch) {
  apsp_ctx *x = (apsp_ctx *)c;
  for (int64_t si = b; si < e; si++)
    bfs_row(x->n, x->indptr, x->indices, x->sources[si], x->out + si * x->n,
            (int32_t *)scratch);
}
void or_apsp_rows(int64_t n, const int64_t *indptr, const int32_t *indices,
                  const int64_t *sources, int64_t nsrc, int32_t *out,
                  int nthreads) {
  apsp_ctx x = {n, indptr, indices, sources, out};
  parallel_for(nthreads, 0, nsrc, 8, sizeof(int32_t) * (size_t)(n + 1), apsp_range, &x);
}

/* ------------------------------------------------------------- partial BFS */
/* _kernels.py:60-131.  Sources [src_begin, src_end); outputs are indexed by
 * (s - src_begin) * k.  Optional work counters: scanned adjacency entries and
 * expanded vertices per source (the TE work unit of SURVEY.md 8(d)). */
static void sort_dist_id(int32_t *nbr, int32_t *dist, int count) {
  /* insertion sort by (dist, id) == argsort of dist*n+id (keys distinct) */
  for (int i = 1; i < count; i++) {
    int32_t a = nbr[i], d = dist[i];
    int j = i - 1;
    while (j >= 0 && (dist[j] > d || (dist[j] == d && nbr[j] > a))) {
      nbr[j + 1] = nbr[j];
      dist[j + 1] = dist[j];
      j--;
    }
    nbr[j + 1] = a;
    dist[j + 1] = d;
  }
}

typedef struct {
  int64_t n;
  const int64_t *indptr;
  const int32_t *indices;
  int32_t k;
  uint64_t seed;
  int64_t src_begin;
  int32_t *nbr_out, *dist_out, *counts_out;
  int64_t *scanned_out, *expanded_out;
} pbfs_ctx;

static void pbfs_range(void *c, int64_t sb, int64_t se, void *scratch) {
  pbfs_ctx *x = (pbfs_ctx *)c;
  const int64_t n = x->n;
  const int64_t *indptr = x->indptr;
  const int32_t *indices = x->indices;
  const int32_t k = x->k;
  /* scratch: stamp | cur | nxt, each n int32; stamp lazily initialised via a
   * per-scratch tag word stored after the three arrays */
  int32_t *stamp = (int32_t *)scratch;
  int32_t *cur = stamp + n;
  int32_t *nxt = cur + n;
  int32_t *inited = nxt + n;
  if (*inited != 0x5eed) {
    for (int64_t i = 0; i < n; i++) stamp[i] = -1;
    *inited = 0x5eed;
  }
  for (int64_t s = sb; s < se; s++) {
    uint64_t state = x->seed + SPLIT_GAMMA * (uint64_t)(s + 1);
    int32_t *a = cur, *b = nxt;
    stamp[s] = (int32_t)s;
    a[0] = (int32_t)s;
    int64_t cur_size = 1;
    int32_t depth = 0;
    int32_t count = 0;
    int64_t scanned = 0, expanded = 0;
    int64_t base = (s - x->src_begin) * (int64_t)k;
    while (count < k && cur_size > 0) {
      int64_t nxt_size = 0;
      for (int64_t ci = 0; ci < cur_size; ci++) {
        int32_t u = a[ci];
        expanded++;
        scanned += indptr[u + 1] - indptr[u];
        for (int64_t p = indptr[u]; p < indptr[u + 1]; p++) {
          int32_t w = indices[p];
          if (stamp[w] != (int32_t)s) {
            stamp[w] = (int32_t)s;
            b[nxt_size++] = w;
          }
        }
      }
      depth += 1;
      if (nxt_size == 0) break;
      int64_t remaining = k - count;
      int64_t take = nxt_size;
      if (nxt_size > remaining) {
        /* random subset of the level that crosses the budget */
        for (int64_t i = 0; i < remaining; i++) {
          int64_t j = i + (int64_t)(sm_next(&state) % (uint64_t)(nxt_size - i));
          int32_t t = b[i];
          b[i] = b[j];
          b[j] = t;
        }
        take = remaining;
      }
      for (int64_t i = 0; i < take; i++) {
        x->nbr_out[base + count + i] = b[i];
        x->dist_out[base + count + i] = depth;
      }
      count += (int32_t)take;
      cur_size = nxt_size;
      int32_t *t = a;
      a = b;
      b = t;
    }
    x->counts_out[s - x->src_begin] = count;
    sort_dist_id(x->nbr_out + base, x->dist_out + base, count);
    if (x->scanned_out) x->scanned_out[s - x->src_begin] = scanned;
    if (x->expanded_out) x->expanded_out[s - x->src_begin] = expanded;
  }
}

void or_partial_bfs_all(int64_t n, const int64_t *indptr,
                        const int32_t *indices, int32_t k, uint64_t seed,
                        int64_t src_begin, int64_t src_end, int32_t *nbr_out,
                        int32_t *dist_out, int32_t *counts_out,
                        int64_t *scanned_out, int64_t *expanded_out,
                        int nthreads) {
  pbfs_ctx x = {n, indptr, indices, k, seed, src_begin, nbr_out, dist_out,
                counts_out, scanned_out, expanded_out};
  size_t bytes = sizeof(int32_t) * (size_t)(3 * n + 1);
  /* scratch is calloc-ed per worker, so the tag word starts at 0 */
  parallel_for(nthreads, src_begin, src_end, 512, bytes, pbfs_range, &x);
}

/* ------------------------------------------------------ numpy SeedSequence */
#define SS_INIT_A 0x43b0d7e5u
#define SS_MULT_A 0x931e8875u
#define SS_INIT_B 0x8b51f9ddu
#define SS_MULT_B 0x58f38dedu
#define SS_MIX_L 0xca01f9ddu
#define SS_MIX_R 0x4973f715u
#define SS_XSHIFT 16

static inline uint32_t ss_hashmix(uint32_t value, uint32_t *hash_const) {
  value ^= *hash_const;
  *hash_const *= SS_MULT_A;
  value *= *hash_const;
  value ^= value >> SS_XSHIFT;
  return value;
}
static inline uint32_t ss_mix(uint32_t x, uint32_t y) {
  uint32_t r = SS_MIX_L * x - SS_MIX_R * y;
  r ^= r >> SS_XSHIFT;
  return r;
}
/* words of a non-negative integer, little-endian; 0 -> [0] */
static int int_words(uint64_t x, uint32_t *w) {
  if (x == 0) {
    w[0] = 0;
    return 1;
  }
  int c = 0;
  while (x) {
    w[c++] = (uint32_t)(x & 0xffffffffu);
    x >>= 32;
  }
  return c;
}
/* SeedSequence(entropy=seed, spawn_key=(key,)).generate_state(4, uint64) */
static void seedseq_state4(uint64_t seed, uint64_t key, uint64_t out[4]) {
  uint32_t ent[8];
  int ne = int_words(seed, ent);
  while (ne < 4) ent[ne++] = 0; /* run entropy padded to pool size when spawn_key */
  uint32_t kw[2];
  int nk = int_words(key, kw);
  for (int i = 0; i < nk; i++) ent[ne++] = kw[i];
  uint32_t pool[4];
  uint32_t hc = SS_INIT_A;
  for (int i = 0; i < 4; i++) pool[i] = ss_hashmix(i < ne ? ent[i] : 0u, &hc);
  for (int s = 0; s < 4; s++)
    for (int d = 0; d < 4; d++)
      if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], &hc));
  for (int s = 4; s < ne; s++)
    for (int d = 0; d < 4; d++) pool[d] = ss_mix(pool[d], ss_hashmix(ent[s], &hc));
  uint32_t st[8];
  uint32_t hb = SS_INIT_B;
  for (int i = 0; i < 8; i++) {
    uint32_t v = pool[i & 3];
    v ^= hb;
    hb *= SS_MULT_B;
    v *= hb;
    v ^= v >> SS_XSHIFT;
    st[i] = v;
  }
  for (int i = 0; i < 4; i++) out[i] = (uint64_t)st[2 * i] | ((uint64_t)st[2 * i + 1] << 32);
}

/* ---------------------------------------------------------------- PCG64 */
typedef struct {
  unsigned __int128 state, inc;
  int has32;
  uint32_t buf32;
} pcg64_t;

static const unsigned __int128 PCG_MULT =
    (((unsigned __int128)0x2360ED051FC65DA4ULL) << 64) | 0x4385DF649FCCF645ULL;

static inline void pcg_step(pcg64_t *r) { r->state = r->state * PCG_MULT + r->inc; }
static inline uint64_t pcg_next64(pcg64_t *r) {
  pcg_step(r);
  uint64_t hi = (uint64_t)(r->state >> 64), lo = (uint64_t)r->state;
  unsigned rot = (unsigned)(r->state >> 122);
  uint64_t x = hi ^ lo;
  return (x >> rot) | (x << ((64 - rot) & 63));
}
static inline uint32_t pcg_next32(pcg64_t *r) {
  if (r->has32) {
    r->has32 = 0;
    return r->buf32;
  }
  uint64_t v = pcg_next64(r);
  r->has32 = 1;
  r->buf32 = (uint32_t)(v >> 32);
  return (uint32_t)(v & 0xffffffffu);
}
static void pcg_seed(pcg64_t *r, const uint64_t s[4]) {
  unsigned __int128 initstate = ((unsigned __int128)s[0] << 64) | s[1];
  unsigned __int128 initseq = ((unsigned __int128)s[2] << 64) | s[3];
  r->state = 0;
  r->inc = (initseq << 1) | 1;
  pcg_step(r);
  r->state += initstate;
  pcg_step(r);
  r->has32 = 0;
  r->buf32 = 0;
}
static uint64_t random_interval(pcg64_t *r, uint64_t max) {
  if (max == 0) return 0;
  uint64_t mask = max, v;
  mask |= mask >> 1;
  mask |= mask >> 2;
  mask |= mask >> 4;
  mask |= mask >> 8;
  mask |= mask >> 16;
  mask |= mask >> 32;
  if (max <= 0xffffffffULL) {
    while ((v = (pcg_next32(r) & mask)) > max) {
    }
  } else {
    while ((v = (pcg_next64(r) & mask)) > max) {
    }
  }
  return v;
}

/* default_rng(SeedSequence(seed, spawn_key=(key,))).permutation(T) into perm */
void or_numpy_permutation(uint64_t seed, uint64_t key, int64_t T, int64_t *perm) {
  uint64_t st[4];
  seedseq_state4(seed, key, st);
  pcg64_t r;
  pcg_seed(&r, st);
  for (int64_t i = 0; i < T; i++) perm[i] = i;
  for (int64_t i = T - 1; i >= 1; i--) {
    int64_t j = (int64_t)random_interval(&r, (uint64_t)i);
    int64_t t = perm[i];
    perm[i] = perm[j];
    perm[j] = t;
  }
}

/* --------------------------------------------------- kNN from a full row */
/* neighbors.py:199-221 for one vertex v.  row: int32 distances (INF32 for
 * unreachable), row[v] is ignored.  Writes up to k (dst, dist) sorted by
 * (dist, id); returns the count.  scratch: >= 2n int64. */
static int knn_select_row(int64_t n, const int32_t *row, int64_t v, int32_t k,
                          uint64_t seed, int32_t *dst, int32_t *dist,
                          int64_t *scratch) {
  int64_t nreach = 0;
  /* histogram-free: find kth by counting per distance (distances < n) */
  int64_t *ids = scratch;          /* reachable ids, ascending */
  int64_t *perm = scratch + n;     /* permutation buffer */
  for (int64_t u = 0; u < n; u++)
    if (u != v && row[u] != INF32) ids[nreach++] = u;
  int cnt = 0;
  if (nreach <= k) {
    for (int64_t i = 0; i < nreach; i++) {
      dst[cnt] = (int32_t)ids[i];
      dist[cnt] = row[ids[i]];
      cnt++;
    }
  } else {
    /* kth smallest value: smallest d such that #{<= d} >= k */
    int32_t lo_d = INF32;
    /* distances are BFS levels; walk levels upward */
    int64_t below = 0;
    int32_t d = 0;
    int32_t maxd = 0;
    for (int64_t i = 0; i < nreach; i++)
      if (row[ids[i]] > maxd) maxd = row[ids[i]];
    int64_t *cntd = (int64_t *)calloc((size_t)maxd + 2, sizeof(int64_t));
    for (int64_t i = 0; i < nreach; i++) cntd[row[ids[i]]]++;
    for (d = 0; d <= maxd; d++) {
      if (below + cntd[d] >= k) {
        lo_d = d;
        break;
      }
      below += cntd[d];
    }
    int64_t T = cntd[lo_d];
    free(cntd);
    int32_t kth = lo_d;
    /* lower (ascending id) then picked ties */
    for (int64_t i = 0; i < nreach; i++)
      if (row[ids[i]] < kth) {
        dst[cnt] = (int32_t)ids[i];
        dist[cnt] = row[ids[i]];
        cnt++;
      }
    int64_t need = k - cnt;
    /* ties ascending id, compacted into ids[] prefix */
    int64_t t = 0;
    for (int64_t i = 0; i < nreach; i++)
      if (row[ids[i]] == kth) ids[t++] = ids[i];
    or_numpy_permutation(seed, (uint64_t)v, T, perm);
    for (int64_t i = 0; i < need; i++) {
      dst[cnt] = (int32_t)ids[perm[i]];
      dist[cnt] = kth;
      cnt++;
    }
  }
  sort_dist_id(dst, dist, cnt);
  return cnt;
}

/* matrix rows -> kNN (neighbors.py:183-237).  out_* are n*k, counts n. */
typedef struct {
  int64_t n;
  const int32_t *matrix;
  const int64_t *indptr;
  const int32_t *indices;
  int32_t k;
  uint64_t seed;
  int64_t src_begin;
  int32_t *out_dst, *out_dist, *counts;
} knn_ctx;

static void knn_matrix_range(void *c, int64_t b, int64_t e, void *scratch) {
  knn_ctx *x = (knn_ctx *)c;
  for (int64_t v = b; v < e; v++)
    x->counts[v] = knn_select_row(x->n, x->matrix + v * x->n, v, x->k, x->seed,
                                  x->out_dst + v * (int64_t)x->k,
                                  x->out_dist + v * (int64_t)x->k,
                                  (int64_t *)scratch);
}

void or_knn_from_matrix(int64_t n, const int32_t *matrix, int32_t k,
                        uint64_t seed, int32_t *out_dst, int32_t *out_dist,
                        int32_t *counts, int nthreads) {
  knn_ctx x = {n, matrix, NULL, NULL, k, seed, 0, out_dst, out_dist, counts};
  parallel_for(nthreads, 0, n, 8, sizeof(int64_t) * (size_t)(2 * n + 2),
               knn_matrix_range, &x);
}

static void full_knn_range(void *c, int64_t b, int64_t e, void *scratch) {
  knn_ctx *x = (knn_ctx *)c;
  int64_t n = x->n;
  int64_t *sc = (int64_t *)scratch;
  int32_t *row = (int32_t *)(sc + 2 * n + 2);
  int32_t *queue = row + n + 1;
  for (int64_t v = b; v < e; v++) {
    bfs_row(n, x->indptr, x->indices, v, row, queue);
    int64_t o = (v - x->src_begin) * (int64_t)x->k;
    x->counts[v - x->src_begin] = knn_select_row(
        n, row, v, x->k, x->seed, x->out_dst + o, x->out_dist + o, sc);
  }
}

/* all_pairs_bfs + knn_from_full_distances fused per source, sources
 * [src_begin, src_end) (outputs indexed from src_begin). */
void or_full_knn(int64_t n, const int64_t *indptr, const int32_t *indices,
                 int32_t k, uint64_t seed, int64_t src_begin, int64_t src_end,
                 int32_t *out_dst, int32_t *out_dist, int32_t *counts,
                 int nthreads) {
  knn_ctx x = {n, NULL, indptr, indices, k, seed, src_begin, out_dst, out_dist, counts};
  size_t bytes = sizeof(int64_t) * (size_t)(2 * n + 2) + sizeof(int32_t) * (size_t)(2 * n + 2);
  parallel_for(nthreads, src_begin, src_end, 4, bytes, full_knn_range, &x);
}

/* ------------------------------------------------------- smooth kNN rho/sigma */
/* numpy pairwise_sum over a contiguous float64 run (loops_utils.h.src). */
static double pairwise_sum(const double *a, int64_t n) {
  if (n < 8) {
    double res = 0.;
    for (int64_t i = 0; i < n; i++) res += a[i];
    return res;
  } else if (n <= 128) {
    double r[8], res;
    int64_t i;
    for (int j = 0; j < 8; j++) r[j] = a[j];
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; j++) r[j] += a[i + j];
    res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res += a[i];
    return res;
  } else {
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pairwise_sum(a, n2) + pairwise_sum(a + n2, n - n2);
  }
}

static double weight_sum(const double *d, int64_t kmax, double rho, double sigma,
                         double *buf) {
  for (int64_t i = 0; i < kmax; i++) buf[i] = exp(-(d[i] - rho) / sigma);
  return pairwise_sum(buf, kmax);
}

/* neighbors.py:261-311 per row.  indptr int64[n+1], dist int32 (CSR rows);
 * kmax = max row count (padding width); target = np.log2(k) from the host.
 * Writes rho[n], sigma[n], and w[nnz] (weights, neighbors.py:309-318). */
typedef struct {
  const int64_t *indptr;
  const int32_t *dist;
  int64_t kmax;
  double target;
  double *rho_out, *sigma_out, *w_out;
} smooth_ctx;

static void smooth_range(void *c, int64_t vb, int64_t ve, void *scratch) {
  const double SMIN = 1e-3, SMAX = 1e3, TOL = 1e-5;
  smooth_ctx *x = (smooth_ctx *)c;
  int64_t kmax = x->kmax;
  double target = x->target;
  double *d = (double *)scratch;
  double *buf = d + kmax + 1;
  for (int64_t v = vb; v < ve; v++) {
    int64_t lo = x->indptr[v], c = x->indptr[v + 1] - lo;
    for (int64_t i = 0; i < kmax; i++) d[i] = i < c ? (double)x->dist[lo + i] : INFINITY;
    double rho = INFINITY;
    for (int64_t i = 0; i < kmax; i++)
      if (d[i] < rho) rho = d[i];
    int all_equal = 1;
    for (int64_t i = 0; i < kmax; i++)
      if (!(isinf(d[i]) || d[i] == rho)) all_equal = 0;
    double sigma = SMAX;
    if (!all_equal) {
      double s_hi = weight_sum(d, kmax, rho, SMAX, buf);
      double s_lo = weight_sum(d, kmax, rho, SMIN, buf);
      int clamp_hi = s_hi < target, clamp_lo = s_lo > target;
      if (clamp_hi) sigma = SMAX;
      if (clamp_lo) sigma = SMIN;
      if (!clamp_hi && !clamp_lo) {
        double los = SMIN, his = SMAX, mid = (los + his) / 2.0;
        int live = 1;
        for (int it = 0; it < 64 && live; it++) {
          double s = weight_sum(d, kmax, rho, mid, buf);
          if (fabs(s - target) < TOL) {
            sigma = mid;
            live = 0;
            break;
          }
          if (s > target)
            his = mid;
          else
            los = mid;
          mid = (los + his) / 2.0;
        }
        if (live) sigma = mid; /* the 65th midpoint (neighbors.py:306-307) */
      }
    }
    x->rho_out[v] = rho;
    x->sigma_out[v] = sigma;
    if (x->w_out)
      for (int64_t i = 0; i < c; i++) x->w_out[lo + i] = exp(-(d[i] - rho) / sigma);
  }
}

void or_smooth_rows(int64_t n, const int64_t *indptr, const int32_t *dist,
                    int64_t kmax, double target, double *rho_out,
                    double *sigma_out, double *w_out, int nthreads) {
  smooth_ctx x = {indptr, dist, kmax, target, rho_out, sigma_out, w_out};
  parallel_for(nthreads, 0, n, 1024, sizeof(double) * (size_t)(2 * kmax + 2),
               smooth_range, &x);
}

/* ------------------------------------------------------- fuzzy union (C1) */
/* neighbors.py:320-350 (and fuzzy_union, 240-242): dedupe each directed row
 * keeping the first occurrence of a destination, then over the union of both
 * orientations h = (a + b) - a*b (a missing orientation counts as 0), exact
 * zeros dropped, keys in (src, dst) order.  Same arithmetic as scipy's
 * w + w.T - w.multiply(w.T) (each entry one add, one multiply, one subtract;
 * -ffp-contract=off), restated per vertex: a row-local sort of the forward
 * row by destination, a counting-sort transpose (in-lists come out in source
 * order) and a merge of the two sorted lists.  oracle.py's numpy
 * fuzzy_union_symmetrize is the slower restatement it is pinned against. */
typedef struct {
  int64_t n;
  const int64_t *indptr;
  const int32_t *dst;
  const double *w;
  int64_t *fptr;   /* deduped forward rows, sorted by destination */
  int32_t *fdst;
  double *fw;
  int64_t *iptr;   /* in-lists (transpose), sorted by source */
  int32_t *isrc;
  double *iw;
  int64_t *optr;   /* output offsets */
  int32_t *osrc, *odst;
  double *ow;
} fu_ctx;

typedef struct {
  int32_t id;
  int64_t pos;
} fu_pair;

static int fu_cmp(const void *a, const void *b) {
  const fu_pair *x = (const fu_pair *)a, *y = (const fu_pair *)b;
  if (x->id != y->id) return x->id < y->id ? -1 : 1;
  return x->pos < y->pos ? -1 : (x->pos > y->pos);
}

/* pass 1: per-row sort + dedupe into a scratch row; count kept entries */
static void fu_rows(void *c, int64_t vb, int64_t ve, void *scratch) {
  fu_ctx *x = (fu_ctx *)c;
  (void)scratch;
  for (int64_t v = vb; v < ve; v++) {
    int64_t lo = x->indptr[v], cnt = x->indptr[v + 1] - lo;
    fu_pair *p = (fu_pair *)malloc(sizeof(fu_pair) * (size_t)(cnt > 0 ? cnt : 1));
    for (int64_t i = 0; i < cnt; i++) {
      p[i].id = x->dst[lo + i];
      p[i].pos = lo + i;
    }
    qsort(p, (size_t)cnt, sizeof(fu_pair), fu_cmp);
    int64_t o = lo, kept = 0;
    for (int64_t i = 0; i < cnt; i++) {
      if (i > 0 && p[i].id == p[i - 1].id) continue; /* keep the first */
      x->fdst[o + kept] = p[i].id;
      x->fw[o + kept] = x->w[p[i].pos];
      kept++;
    }
    x->fptr[v] = kept; /* count; turned into the row length below */
    free(p);
  }
}

static int64_t fu_merge_row(const fu_ctx *x, int64_t v, int write) {
  int64_t a0 = x->indptr[v], an = a0 + x->fptr[v];
  int64_t b0 = x->iptr[v], bn = x->iptr[v + 1];
  int64_t o = write ? x->optr[v] : 0, kept = 0;
  while (a0 < an || b0 < bn) {
    int32_t id;
    double a = 0.0, b = 0.0;
    if (b0 >= bn || (a0 < an && x->fdst[a0] < x->isrc[b0])) {
      id = x->fdst[a0];
      a = x->fw[a0++];
    } else if (a0 >= an || x->isrc[b0] < x->fdst[a0]) {
      id = x->isrc[b0];
      b = x->iw[b0++];
    } else {
      id = x->fdst[a0];
      a = x->fw[a0++];
      b = x->iw[b0++];
    }
    double s = a + b;
    double pr = a * b;
    double h = s - pr;
    if (h != 0.0) {
      if (write) {
        x->osrc[o + kept] = (int32_t)v;
        x->odst[o + kept] = id;
        x->ow[o + kept] = h;
      }
      kept++;
    }
  }
  return kept;
}

static void fu_count(void *c, int64_t vb, int64_t ve, void *scratch) {
  fu_ctx *x = (fu_ctx *)c;
  (void)scratch;
  for (int64_t v = vb; v < ve; v++) x->optr[v + 1] = fu_merge_row(x, v, 0);
}

static void fu_write(void *c, int64_t vb, int64_t ve, void *scratch) {
  fu_ctx *x = (fu_ctx *)c;
  (void)scratch;
  for (int64_t v = vb; v < ve; v++) fu_merge_row(x, v, 1);
}

/* Returns E (the number of symmetrised directed edges).  Call twice: with
 * osrc == NULL to size, then with outputs of E entries (nbr_indptr n+1).
 * The scratch arrays are rebuilt on each call (oracle: simplicity first). */
int64_t or_fuzzy_union(int64_t n, const int64_t *indptr, const int32_t *dst,
                       const double *w, int32_t *osrc, int32_t *odst, double *ow,
                       int64_t *nbr_indptr, int nthreads) {
  int64_t nnz = indptr[n];
  fu_ctx x;
  memset(&x, 0, sizeof(x));
  x.n = n;
  x.indptr = indptr;
  x.dst = dst;
  x.w = w;
  x.fptr = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
  x.fdst = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nnz + 1));
  x.fw = (double *)malloc(sizeof(double) * (size_t)(nnz + 1));
  parallel_for(nthreads, 0, n, 4096, 0, fu_rows, &x);
  /* transpose: in-list of d gets (v, w) for every kept forward (v, d) */
  x.iptr = (int64_t *)calloc((size_t)n + 2, sizeof(int64_t));
  for (int64_t v = 0; v < n; v++)
    for (int64_t i = indptr[v]; i < indptr[v] + x.fptr[v]; i++) x.iptr[x.fdst[i] + 1]++;
  for (int64_t v = 0; v < n; v++) x.iptr[v + 1] += x.iptr[v];
  x.isrc = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nnz + 1));
  x.iw = (double *)malloc(sizeof(double) * (size_t)(nnz + 1));
  int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
  memcpy(fill, x.iptr, sizeof(int64_t) * (size_t)(n + 1));
  for (int64_t v = 0; v < n; v++) /* v ascending: in-lists in source order */
    for (int64_t i = indptr[v]; i < indptr[v] + x.fptr[v]; i++) {
      int64_t d = x.fdst[i];
      x.isrc[fill[d]] = (int32_t)v;
      x.iw[fill[d]] = x.fw[i];
      fill[d]++;
    }
  free(fill);
  x.optr = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
  parallel_for(nthreads, 0, n, 4096, 0, fu_count, &x);
  for (int64_t v = 0; v < n; v++) x.optr[v + 1] += x.optr[v];
  int64_t E = x.optr[n];
  if (osrc) {
    x.osrc = osrc;
    x.odst = odst;
    x.ow = ow;
    parallel_for(nthreads, 0, n, 4096, 0, fu_write, &x);
    if (nbr_indptr) memcpy(nbr_indptr, x.optr, sizeof(int64_t) * (size_t)(n + 1));
  }
  free(x.fptr);
  free(x.fdst);
  free(x.fw);
  free(x.iptr);
  free(x.isrc);
  free(x.iw);
  free(x.optr);
  return E;
}

/* ------------------------------------------------------------------- SGD */
static inline double clip4(double x) {
  if (x > 4.0) return 4.0;
  if (x < -4.0) return -4.0;
  return x;
}
static inline int is_neighbor(const int64_t *ip, const int32_t *ix, int64_t u,
                              int64_t c) {
  int64_t lo = ip[u], hi = ip[u + 1];
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2; /* lo, hi >= 0: floor division == C division */
    if (ix[mid] < c)
      lo = mid + 1;
    else if (ix[mid] > c)
      hi = mid;
    else
      return 1;
  }
  return 0;
}

/* _kernels.py:158-223.  coords float64 (n,2) in place; state in/out.
 * neg_log (len(order)*n_neg, may be NULL): accepted negative or -1.
 * theta_log (same shape, may be NULL): theta drawn for coincident points, NaN
 * otherwise. */
void or_sgd_sweep(double *coords, int64_t n, const int32_t *e_src,
                  const int32_t *e_dst, const double *e_w, const int64_t *order,
                  int64_t n_order, const int64_t *nbr_indptr,
                  const int32_t *nbr_indices, double a, double b, double lr,
                  int32_t n_neg, uint64_t *state_io, int32_t *neg_log,
                  double *theta_log) {
  uint64_t state = *state_io;
  for (int64_t i = 0; i < n_order; i++) {
    int64_t e = order[i];
    int64_t u = e_src[e], v = e_dst[e];
    double h = e_w[e];
    double dx = coords[2 * u] - coords[2 * v];
    double dy = coords[2 * u + 1] - coords[2 * v + 1];
    double d2 = dx * dx + dy * dy;
    if (d2 > 0.0) {
      double pb = pow(d2, b);
      double g = -2.0 * a * b * h * (pb / d2) / (a * pb + 1.0);
      double gx = clip4(g * dx), gy = clip4(g * dy);
      coords[2 * u] += lr * gx;
      coords[2 * u + 1] += lr * gy;
      coords[2 * v] -= lr * gx;
      coords[2 * v + 1] -= lr * gy;
    }
    for (int q = 0; q < n_neg; q++) {
      int64_t slot = i * (int64_t)n_neg + q;
      int64_t c = -1;
      for (int t = 0; t < 8; t++) {
        int64_t cand = (int64_t)(sm_next(&state) % (uint64_t)n);
        if (cand == u) continue;
        if (!is_neighbor(nbr_indptr, nbr_indices, u, cand)) {
          c = cand;
          break;
        }
      }
      if (neg_log) neg_log[slot] = (int32_t)c;
      if (theta_log) theta_log[slot] = NAN;
      if (c < 0) continue;
      double ddx = coords[2 * u] - coords[2 * c];
      double ddy = coords[2 * u + 1] - coords[2 * c + 1];
      double dd2 = ddx * ddx + ddy * ddy;
      double gx, gy;
      if (dd2 > 0.0) {
        double g = 2.0 * b / ((0.001 + dd2) * (a * pow(dd2, b) + 1.0));
        gx = clip4(g * ddx);
        gy = clip4(g * ddy);
      } else {
        double theta = sm_next_float(&state) * 6.283185307179586;
        if (theta_log) theta_log[slot] = theta;
        gx = 4.0 * cos(theta);
        gy = 4.0 * sin(theta);
      }
      coords[2 * u] += lr * gx;
      coords[2 * u + 1] += lr * gy;
    }
  }
  *state_io = state;
}

/* Replay of one sweep with supplied negatives (-1 = skipped slot) and thetas
 * (used when the replayed pair is coincident). Same arithmetic as above. */
void or_sgd_replay(double *coords, const int32_t *e_src, const int32_t *e_dst,
                   const double *e_w, const int64_t *order, int64_t n_order,
                   const int32_t *negs, const double *thetas, double a, double b,
                   double lr, int32_t n_neg) {
  for (int64_t i = 0; i < n_order; i++) {
    int64_t e = order[i];
    int64_t u = e_src[e], v = e_dst[e];
    double h = e_w[e];
    double dx = coords[2 * u] - coords[2 * v];
    double dy = coords[2 * u + 1] - coords[2 * v + 1];
    double d2 = dx * dx + dy * dy;
    if (d2 > 0.0) {
      double pb = pow(d2, b);
      double g = -2.0 * a * b * h * (pb / d2) / (a * pb + 1.0);
      double gx = clip4(g * dx), gy = clip4(g * dy);
      coords[2 * u] += lr * gx;
      coords[2 * u + 1] += lr * gy;
      coords[2 * v] -= lr * gx;
      coords[2 * v + 1] -= lr * gy;
    }
    for (int q = 0; q < n_neg; q++) {
      int64_t slot = i * (int64_t)n_neg + q;
      int64_t c = negs[slot];
      if (c < 0) continue;
      double ddx = coords[2 * u] - coords[2 * c];
      double ddy = coords[2 * u + 1] - coords[2 * c + 1];
      double dd2 = ddx * ddx + ddy * ddy;
      double gx, gy;
      if (dd2 > 0.0) {
        double g = 2.0 * b / ((0.001 + dd2) * (a * pow(dd2, b) + 1.0));
        gx = clip4(g * ddx);
        gy = clip4(g * ddy);
      } else {
        double theta = thetas[slot];
        gx = 4.0 * cos(theta);
        gy = 4.0 * sin(theta);
      }
      coords[2 * u] += lr * gx;
      coords[2 * u + 1] += lr * gy;
    }
  }
}

int or_max_threads(void) { return (int)sysconf(_SC_NPROCESSORS_ONLN); }
