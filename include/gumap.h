/*
 * gumap.h -- C ABI of libgumap.so, the B200 (sm_100a) hot path of the
 * graph_umap layouts (GUMAP / SS / SL / SSSL, arXiv 2509.19703).
 *
 * Conventions
 *   - Plain pointers and sizes only.  Array arguments are DEVICE pointers
 *     unless the name starts with host_.  `stream` is a cudaStream_t (NULL =
 *     legacy default stream).  Every call is asynchronous on `stream` unless
 *     documented otherwise.
 *   - Return value: 0 = ok; 1 = bad argument; 2 = CUDA error; 3 = workspace too
 *     small; 4 = unsupported input.  gu_last_error() gives the message.  The
 *     Python layer maps these to the reference's exceptions (ValueError etc.).
 *   - CSR graphs use int32 row offsets (2m < 2^31, every BASELINE config) and
 *     int32 neighbour ids sorted ascending per row, as graph_umap's Graph
 *     (graph.py:16-71) after the int64 -> int32 offset narrowing done by the
 *     device CSR store.
 *   - Caller-owned outputs, fixed stride k per source ("records"), as the
 *     reference's numba kernels write them (_kernels.py:61 nbr_out/dist_out/
 *     counts_out).
 *
 * Each entry point cites the reference interface it replaces
 * (/root/reference/pkg/src/graph_umap/...).
 */
#ifndef GUMAP_H
#define GUMAP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------ library */
int gu_version(void);                 /* ABI version, currently 1 */
const char* gu_last_error(void);      /* thread-local message of the last failure */
int gu_device_sync(void* stream);     /* cudaStreamSynchronize + error check */
int gu_host_is_pinned(const void* p); /* 1 if p lies in page-locked host memory */

/* ---------------------------------------------- C0+C1 partial BFS-kNN
 * Replaces _kernels.py:60-131 partial_bfs_all(indptr, indices, k, seed,
 * nbr_out, dist_out, counts_out), reached via neighbors.py:137 partial_bfs.
 * indptr / indices: the CSR the reference's Graph holds (graph.py:16-71) --
 * the SYMMETRIC adjacency of an undirected simple graph, rows sorted
 * ascending; the hub tier tests "x in N(H)" as "H in N(x)".
 * Sources [src_begin, src_end); row r = s - src_begin of out_nbr/out_dist
 * (stride k) holds the k hop-nearest others of s sorted by (dist, id), ties at
 * the crossing level chosen by the reference's splitmix64 partial
 * Fisher-Yates.  out_count[r] < k only when the component is smaller.
 * work_counters (nullable, 2 x uint64): adjacency entries scanned and vertices
 * expanded, summed over sources (the TE work unit).
 * tier2_warps: per-warp n-int scratch slots for sources whose BFS ball exceeds
 * the shared-memory tiers; workspace size from gu_partial_bfs_workspace_size. */
size_t gu_partial_bfs_workspace_size(int64_t n, int64_t nsrc, int32_t tier2_warps);
int gu_partial_bfs_knn(int64_t n, const int32_t* indptr, const int32_t* indices,
                       int32_t k, uint64_t seed, int64_t src_begin, int64_t src_end,
                       int32_t* out_nbr, int32_t* out_dist, int32_t* out_count,
                       uint64_t* work_counters, void* workspace, size_t ws_bytes,
                       int32_t tier2_warps, void* stream);
/* synchronous: sources that left the register tier F, that reached the
 * big-ball tier (C / 1b) and that reached tier 2 in the last call on this
 * workspace (3 ints) */
int gu_partial_bfs_overflow_counts(void* workspace, int64_t nsrc, int32_t* host_out3);
/* synchronous: sources that left tier F (to 1a), tier 1a (to the hub tier H),
 * tier H (to tier C / 1b) and tier C / 1b (to tier 2) in the last call on
 * this workspace (4 ints) */
int gu_partial_bfs_tier_counts(void* workspace, int64_t nsrc, int32_t* host_out4);

/* ----------------------------------------------- C0 full BFS (bitset)
 * Replaces _kernels.py:33-57 apsp_rows via neighbors.py:120 all_pairs_bfs:
 * int32 hop-distance rows for sources [src_begin, src_end) into out_rows
 * (row r = s - src_begin, n entries, INT32_MAX = unreachable).  64 sources per
 * bitset word, level-synchronous. */
size_t gu_full_bfs_workspace_size(int64_t n, int32_t k, int32_t batches_in_flight);
int gu_apsp_rows(int64_t n, const int32_t* indptr, const int32_t* indices,
                 int64_t src_begin, int64_t src_end, int32_t* out_rows,
                 void* workspace, size_t ws_bytes, int32_t batches_in_flight,
                 void* stream);

/* ----------------------------------------------- C0+C1 full BFS-kNN fused
 * Replaces all_pairs_bfs (neighbors.py:120) + knn_from_full_distances
 * (neighbors.py:183-237) without materialising the n x n matrix: bitset BFS
 * with per-source early exit at the k-th distance, k-th distance ties chosen
 * by numpy's SeedSequence(seed, spawn_key=(v,)) -> PCG64 -> permutation
 * restated on device.  Records as gu_partial_bfs_knn.
 * work_counters: adjacency entries scanned (TE) and BFS levels run. */
int gu_full_bfs_knn(int64_t n, const int32_t* indptr, const int32_t* indices,
                    int32_t k, uint64_t seed, int64_t src_begin, int64_t src_end,
                    int32_t* out_nbr, int32_t* out_dist, int32_t* out_count,
                    uint64_t* work_counters, void* workspace, size_t ws_bytes,
                    int32_t batches_in_flight, void* stream);

/* kNN selection from explicit int32 distance rows (neighbors.py:199-221), for
 * SparseDistanceSet objects that arrive with a materialised matrix.
 * rows: nrows x n (row r belongs to vertex row_begin + r).  scratch: 2*n int32
 * per warp slot (gu_knn_from_rows_workspace_size). */
size_t gu_knn_from_rows_workspace_size(int64_t n, int32_t slots);
int gu_knn_from_rows(int64_t n, const int32_t* rows, int64_t row_begin, int64_t nrows,
                     int32_t k, uint64_t seed, int32_t* out_nbr, int32_t* out_dist,
                     int32_t* out_count, void* workspace, size_t ws_bytes,
                     int32_t slots, void* stream);

/* ---------------------------------------------------- record packing
 * Fixed-stride records -> CSR (neighbors.py:166-175, the Python packing loop
 * the reference runs per vertex).  out_indptr int64[nrows+1]. */
int gu_pack_records(int64_t nrows, int32_t k, const int32_t* rec_nbr,
                    const int32_t* rec_dist, const int32_t* rec_count,
                    int64_t* out_indptr, int32_t* out_dst, int32_t* out_dist,
                    void* workspace, size_t ws_bytes, void* stream);
size_t gu_pack_records_workspace_size(int64_t nrows);

/* --------------------------------------------------- C1 smooth kNN rho/sigma
 * Replaces neighbors.py:261-318: rho = row min, sigma by the reference's
 * 64-step bisection on [1e-3, 1e3] (tol 1e-5, numpy pairwise row sums over
 * rows padded to kmax, non-converged rows take the next midpoint), weights
 * w = exp(-(d - rho) / sigma).  target = np.log2(k) computed by the caller.
 * workspace: gu_smooth_knn_workspace_size(n) bytes (0 below 4096 rows), the
 * memoised-sigma profile table and per-row slots of this call alone: calls
 * on different streams are independent. */
size_t gu_smooth_knn_workspace_size(int64_t n);
int gu_smooth_knn(int64_t n, const int64_t* indptr, const int32_t* dist, int32_t kmax,
                  double target, double* rho, double* sigma, double* w, void* workspace,
                  size_t ws_bytes, void* stream);

/* ----------------------------------------------- C1 fuzzy-union symmetrise
 * Replaces neighbors.py:320-350 (dedupe first occurrence, w + w^T - w o w^T
 * with exact zeros dropped, lexsort by (src, dst), CSR neighbour lookup).
 * Outputs have capacity 2*nnz; *host_E receives the edge count (synchronous).
 * nbr_indptr int64[n+1]; nbr_indices == sym_dst (callers may alias). */
size_t gu_symmetrize_workspace_size(int64_t n, int64_t nnz);
int gu_symmetrize(int64_t n, int64_t nnz, const int64_t* indptr, const int32_t* dst,
                  const double* w, int32_t* sym_src, int32_t* sym_dst, double* sym_w,
                  int64_t* nbr_indptr, int64_t* host_E, void* workspace,
                  size_t ws_bytes, void* stream);
/* The same call for weights that gu_smooth_knn just produced: smooth_workspace
 * is that call's workspace (same n, untouched since).  The backward side of
 * the union then reads each weight from the memoised per-profile table in it
 * instead of gathering w[] in destination order -- identical output.  A null
 * or short smooth_workspace makes it gu_symmetrize. */
int gu_symmetrize_memo(int64_t n, int64_t nnz, const int64_t* indptr, const int32_t* dst,
                       const double* w, int32_t* sym_src, int32_t* sym_dst, double* sym_w,
                       int64_t* nbr_indptr, int64_t* host_E, void* workspace, size_t ws_bytes,
                       const void* smooth_workspace, size_t smooth_ws_bytes, void* stream);

/* ---------------------------------------------------- C2 SGD (Hogwild fp32)
 * The layout epochs of layout.py:314-360 / sgd_sweep (_kernels.py:158-223)
 * with the same per-visit semantics (attraction on both ends scaled by h,
 * n_neg rejection-sampled repulsions of the head against non-neighbours,
 * 8 draws max, per-component clip +-4, random direction for coincident
 * points), run as a Hogwild epoch over fp32 float2 coordinates.  The epoch
 * schedule (fresh order per epoch, or a sliding window of `window` edges over
 * one shuffled order) and the negatives come from a counter-based 64-bit hash
 * keyed by seed.
 * edges: int4 records {src, dst, float-bits(h), (row start << 6) | degree or -1},
 * built in a shuffled order by gu_sgd_prepare_edges (perm_out, nullable,
 * receives the sym edge id of every record position).  nbr CSR int32.
 * Runs epochs [epoch_begin, epoch_end) of a t-epoch schedule,
 * lr_e = lr0 * (1 - e/t).  diverged (int32, device): atomicMin'd with the
 * first epoch that produced a non-finite coordinate (init to INT32_MAX).
 * concurrency: maximum number of edge visits in flight (threads); 0 = fill
 * the GPU.  Hogwild stays statistically close to the sequential sweep only
 * while concurrency << n, so callers cap it for small graphs.
 * nbr_filter (nullable): per-vertex 64-bit Bloom words of the neighbour ids
 * (2 hash bits per id) from gu_sgd_neighbor_filter (8 bytes x n); a negative
 * with a clear bit skips the row search (exact: a hit still searches). */
/* Edge-record layout for a concurrency cap: 32 bytes (the record carries
 * its head's filter; GPU-filling epochs) or 16 bytes (the 64-bit table of
 * gu_sgd_neighbor_filter is gathered; small caps). */
int32_t gu_sgd_record_bytes_for(int64_t concurrency);
/* record_mode: 0 = 16-byte records + table, 1 = 32-byte records with the
 * head's 128-bit Bloom word, 2 = 32-byte records with [min, max] of the
 * head's neighbour ids and its 64-bit word (for ids in a locality order,
 * gu_bfs_order).  relabel (nullable): old id -> new id; nbr_indptr /
 * nbr_indices are then the neighbour CSR in the new ids. */
int gu_sgd_prepare_edges(int64_t E, const int32_t* sym_src, const int32_t* sym_dst,
                         const double* sym_w, const int32_t* nbr_indptr,
                         const int32_t* nbr_indices, const int32_t* relabel, int32_t record_mode,
                         uint64_t seed, void* edges, int32_t* perm_out, void* stream);
/* REC_RANGE records (record_mode 2) in a local stored order: the edges in
 * the order of the relabelled neighbour CSR (new_indptr / new_indices from
 * gu_bfs_order), shuffled inside blocks of `block` consecutive edges, so an
 * epoch tile touches nearby vertices; perm_out maps positions to the sym edge
 * ids of the caller's CSR (nbr_indptr / nbr_indices, rows sorted). */
int gu_sgd_prepare_edges_local(int64_t n, int64_t E, const double* sym_w,
                               const int32_t* new_indptr, const int32_t* new_indices,
                               const int32_t* order, const int32_t* nbr_indptr,
                               const int32_t* nbr_indices, int64_t block, uint64_t seed,
                               void* edges, int32_t* perm_out, void* stream);
/* Locality order of a symmetric graph for the SGD epochs (csrc/order.cu):
 * vertices sorted by (BFS level from a pseudo-peripheral vertex, id), the
 * unreached last.  order[new] = old, perm[old] = new; new_indptr /
 * new_indices (nullable) receive the graph in the new ids (rows sorted);
 * host_levels[2] the depths of the two BFS sweeps.  Synchronous. */
size_t gu_bfs_order_workspace_size(int64_t n, int64_t m);
int gu_bfs_order(int64_t n, const int32_t* indptr, const int32_t* indices, int32_t* order,
                 int32_t* perm, int32_t* new_indptr, int32_t* new_indices, int32_t* host_levels,
                 void* workspace, size_t ws_bytes, void* stream);
/* numpy.random.default_rng(seed).uniform(low, high, count) (PCG64 seeded by
 * SeedSequence(seed), numpy's next_double and random_uniform), bit-exact, into
 * device float64 out[count]; replaces random_init's draws (layout.py:307-311)
 * for large n. */
int gu_random_uniform(int64_t count, uint64_t seed, double low, double high, double* out,
                      void* stream);
int gu_sgd_neighbor_filter(int64_t n, const int32_t* nbr_indptr, const int32_t* nbr_indices,
                           void* filter_out, void* stream);
/* Exact neighbour sets for small concurrency caps (record_mode 3): vertex u's
 * neighbour ids in a table of S_u = next_pow2(4 deg(u)) >= 4 int32 slots
 * (empty = -1) at table[off[u] ..), probed in buckets of 4 slots (16 bytes).  _layout writes off (int32[n+1],
 * exclusive sums of S_u) and the total slot count to *host_slots
 * (synchronous; GU_ERR_UNSUPPORTED when a row exceeds 8192 ids or the total
 * 2^28 slots); gu_sgd_neighbor_hash fills the table (`slots` int32).  The
 * table is then the nbr_filter argument of gu_sgd_epochs for record_mode 3,
 * whose records come from gu_sgd_prepare_edges_hash: {src, dst,
 * float-bits(h), off[src] << 4 | log2 S_src} in the shuffled order. */
int gu_sgd_neighbor_hash_layout(int64_t n, const int32_t* nbr_indptr, int32_t* off,
                                int64_t* host_slots, void* stream);
int gu_sgd_neighbor_hash(int64_t n, const int32_t* nbr_indptr, const int32_t* nbr_indices,
                         const int32_t* off, int32_t* table, int64_t slots, void* stream);
int gu_sgd_prepare_edges_hash(int64_t E, const int32_t* sym_src, const int32_t* sym_dst,
                              const double* sym_w, const int32_t* off, uint64_t seed, void* edges,
                              int32_t* perm_out, void* stream);
int gu_sgd_epochs(int64_t n, int64_t E, float* coords_xy, const void* edges,
                  int32_t record_mode, const int32_t* nbr_indptr, const int32_t* nbr_indices,
                  const void* nbr_filter, float a, float b,
                  float lr0, int32_t t, int32_t epoch_begin, int32_t epoch_end,
                  int32_t n_neg, int64_t window, int32_t windowed, uint64_t seed,
                  int64_t concurrency, int32_t* diverged, void* stream);
/* Opt-in deterministic epochs (sequential by default, parallel
 * modes only statistically reproducible -- this mode restores bitwise
 * repeatability, acceptance criterion 9).  Same visits, draws and update
 * rule as gu_sgd_epochs, run in batches of `batch` visits: a batch reads
 * the positions as they stood when it started and adds its deltas as
 * 2^-32 fixed-point integers into acc (int64[2n], zero on entry, zero on
 * return), applied after the batch -- integer sums do not depend on the
 * order the atomics land in.  Replaces the same _run_sgd loop as
 * gu_sgd_epochs (layout.py:314-360). */
int gu_sgd_epochs_deterministic(int64_t n, int64_t E, float* coords_xy, const void* edges,
                                int32_t record_mode, const int32_t* nbr_indptr,
                                const int32_t* nbr_indices,
                                const void* nbr_filter, float a, float b, float lr0, int32_t t,
                                int32_t epoch_begin, int32_t epoch_end, int32_t n_neg,
                                int64_t window, int32_t windowed, uint64_t seed, int64_t batch,
                                int64_t* acc, int32_t* diverged, void* stream);
/* positions visited by epoch `epoch` (visit_log): window/permutation indices
 * into the prepared edge array, length window (windowed) or E (full). */
int gu_sgd_visit_order(int64_t E, int32_t epoch, int64_t window, int32_t windowed,
                       uint64_t seed, int64_t* out_order, void* stream);

/* ----------------------------------------- C2 order-faithful replay (fp64)
 * Parity check (b): replays one sgd_sweep (_kernels.py:158-223) in float64
 * with a supplied visit order, accepted negatives (-1 = skipped slot) and
 * thetas (used for coincident pairs).  Host-side wave schedule
 * (gu_replay_schedule, synchronous, host pointers) groups visits into
 * conflict-free waves; the device applies the waves in order, so the result
 * equals the sequential sweep up to libm-vs-CUDA pow/cos/sin ulps. */
int gu_replay_schedule(int64_t n, int64_t n_order, const int32_t* host_src,
                       const int32_t* host_dst, const int64_t* host_order,
                       const int32_t* host_negs, int32_t n_neg, int64_t* host_wave_items,
                       int64_t* host_wave_offsets, int64_t* host_n_waves);
int gu_sgd_replay_f64(int64_t n, double* coords, const int32_t* e_src, const int32_t* e_dst,
                      const double* e_w, const int64_t* order, const int32_t* negs,
                      const double* thetas, int32_t n_neg, double a, double b, double lr,
                      const int64_t* wave_items, const int64_t* wave_offsets,
                      int64_t n_waves, void* stream);


/* ----------------------------------------- layout-quality metrics (8(f) 1)
 * Restate metrics.py:41-190 on the GPU.  coords_xy: float64 (n, 2) row-major.
 * gu_stress: both passes of metrics.py:106-131 fused into the 64-source bitset
 * BFS (no hop rows in memory); out3 (device, 3 doubles) = (sum of the stress
 * terms, scale, unreachable flag); stress = out3[0] / (n*n - n).  sources
 * (nullable, nsources distinct ids): only those rows -- the sampled estimator
 * (scale fitted on the same pairs), stress = out3[0] / (nsources * (n - 1)). */
size_t gu_stress_workspace_size(int64_t n);
int gu_stress(int64_t n, const int32_t* indptr, const int32_t* indices,
              const double* coords_xy, int32_t rescale, const int32_t* sources,
              int64_t nsources, double* out3, void* workspace, size_t ws_bytes, void* stream);
/* count_crossings (metrics.py:176-190, _kernels.py:244-296): exact count of
 * unordered edge pairs (edges int32 (m, 2)) whose open segments cross.
 * gu_crossings_grid writes a g x g square grid over the coordinates' bounding
 * box into grid_out (gu_grid_bytes); gu_crossings_incidences gives per-edge
 * cell counts (int64[m]) whose sum n_inc sizes gu_crossings' workspace;
 * out_count: device uint64. */
size_t gu_grid_bytes(void);
int gu_crossings_grid(int64_t n, const double* coords_xy, int32_t g, void* grid_out,
                      void* stream);
int gu_crossings_incidences(int64_t m, const int32_t* edges, const double* coords_xy,
                            const void* grid, int64_t* out_counts, void* stream);
size_t gu_crossings_workspace_size(int64_t m, int64_t n_inc, int32_t g);
int gu_crossings(int64_t m, const int32_t* edges, const double* coords_xy, const void* grid,
                 int32_t g, int64_t n_inc, uint64_t* out_count, void* workspace,
                 size_t ws_bytes, void* stream);
/* neighborhood_preservation (metrics.py:41-79): out_sum (device double) = the
 * sum over v of |ball_r(v) & nearest_q(v)| / |union| -- over every vertex,
 * or over the nsources distinct vertices of `sources` (nullable; the sampled
 * estimator); the caller divides.  slots = concurrent warps, each with 2n
 * ints of scratch. */
size_t gu_np_workspace_size(int64_t n, int32_t slots);
int gu_neighborhood_preservation(int64_t n, const int32_t* indptr, const int32_t* indices,
                                 const double* coords_xy, int32_t r, int32_t slots,
                                 const int32_t* sources, int64_t nsources, double* out_sum,
                                 void* workspace, size_t ws_bytes, void* stream);


/* ------------------------------------------- spectral_init (8(f) row 2)
 * layout.py:221-304.  gu_spectral_degree: inv_sqrt = deg^-1/2, sqrt_deg.
 * gu_spectral_op: y = P (x' + D^-1/2 A D^-1/2 x'), x' = P x, P = I - B B^T,
 * the deflated 2I - L_sym of layout.py:270-273; basis: nb <= 4 orthonormal
 * float64 columns (column j at basis + j*n); x != y. */
int gu_spectral_degree(int64_t n, const int32_t* indptr, double* inv_sqrt, double* sqrt_deg,
                       void* stream);
size_t gu_spectral_op_workspace_size(int64_t n);
int gu_spectral_op(int64_t n, const int32_t* indptr, const int32_t* indices,
                   const double* inv_sqrt, const double* basis, int32_t nb, const double* x,
                   double* y, void* workspace, size_t ws_bytes, void* stream);
/* Thick-restart Lanczos steps of spectral_init's eigensolver
 * (layout.py:275-278 eigsh k=1 'LM', ncv=32, tol=1e-6, on the operator
 * above): gu_lanczos_prepare computes vb = B^T v and the operator input of v;
 * gu_lanczos_step(j) applies the operator to row j of V ((ncv+1) x n), runs
 * two classical Gram-Schmidt passes against [B; V_0..V_j] with the dots fused
 * into the passes, and writes row j+1 of V, row j+1 of VB ((ncv+1) x 4 rows
 * V_i^T B) and H[:j+2, j] ((ncv+1) x ncv).  No host synchronisation. */
size_t gu_lanczos_workspace_size(int64_t n);
int gu_lanczos_prepare(int64_t n, const double* inv_sqrt, const double* basis, int32_t nb,
                       const double* v, double* vb, void* workspace, size_t ws_bytes,
                       void* stream);
int gu_lanczos_step(int64_t n, const int32_t* indptr, const int32_t* indices,
                    const double* inv_sqrt, const double* basis, int32_t nb, double* V,
                    double* VB, double* H, int32_t ncv, int32_t j, void* workspace,
                    size_t ws_bytes, void* stream);

/* ------------------------------------------------- connected components
 * graph.py is_connected / largest_connected_component: labels[v] = smallest
 * vertex id of v's component (lock-free union-find); out_ncomp: device int. */
size_t gu_components_workspace_size(int64_t n);
int gu_connected_components(int64_t n, const int32_t* indptr, const int32_t* indices,
                            int32_t* labels, int32_t* out_ncomp, void* workspace,
                            size_t ws_bytes, void* stream);


/* -------------------------------------- spectral sparsifier (8(f) row 3)
 * sparsify.py:49-205.  gu_resistance_exact_gather: r_e from the grounded
 * Laplacian inverse X ((n-1)^2 float64, vertex 0 grounded).
 * gu_resistance_sketch: q counter-based Rademacher projections of the
 * incidence matrix, block Jacobi-PCG (rtol, maxiter), out_r[e] = sum_i
 * (y_i[u] - y_i[v])^2; status 4 = not converged (host_resid = residual).
 * gu_sparsify_select: keep[e] (device uint8, by edge id) = max-resistance
 * spanning tree + the first (target - tree) non-tree edges by (-r, u, v). */
int gu_resistance_exact_gather(int64_t m, const int32_t* edges, const double* X, int64_t n,
                               double* out_r, void* stream);
size_t gu_resistance_sketch_workspace_size(int64_t n, int32_t q);
int gu_resistance_sketch(int64_t n, const int32_t* indptr, const int32_t* indices, int64_t m,
                         const int32_t* edges, int32_t q, uint64_t seed, double rtol,
                         int32_t maxiter, double* out_r, int32_t* host_iters,
                         double* host_resid, void* workspace, size_t ws_bytes, void* stream);
size_t gu_sparsify_workspace_size(int64_t n, int64_t m);
int gu_sparsify_select(int64_t n, int64_t m, const int32_t* edges, const double* r,
                       int64_t target, uint8_t* keep, int32_t* host_tree_edges,
                       void* workspace, size_t ws_bytes, void* stream);


/* ------------------------------------ graph construction / LCC (8(f) 4)
 * graph.py:114-232.  gu_build_graph_ids: raw int64 (npairs, 2) ids on the
 * device -> host_out = (n, canonical edge count m, self loops dropped);
 * gu_build_graph_csr (same workspace): sorted unique ids (int64 n), edges
 * (int64 (m, 2), (u, v) order), indptr (int64 n+1), indices (int32 2m).
 * gu_lcc_plan: host_out = (components, champion size n2, its edges m2);
 * gu_lcc_build: old id of each kept vertex (int32 n2), edges, CSR. */
size_t gu_build_graph_workspace_size(int64_t npairs);
int gu_build_graph_ids(int64_t npairs, const int64_t* raw, int64_t* host_out, void* workspace,
                       size_t ws_bytes, void* stream);
int gu_build_graph_csr(int64_t npairs, int64_t n, int64_t m, int64_t* out_ids,
                       int64_t* out_edges, int64_t* out_indptr, int32_t* out_indices,
                       void* workspace, size_t ws_bytes, void* stream);
size_t gu_lcc_workspace_size(int64_t n, int64_t m);
int gu_lcc_plan(int64_t n, int64_t m, const int32_t* indptr, const int32_t* indices,
                const int64_t* edges, int64_t* host_out, void* workspace, size_t ws_bytes,
                void* stream);
int gu_lcc_build(int64_t n, int64_t m, int64_t n2, int64_t m2, int32_t* out_old_ids,
                 int64_t* out_edges, int64_t* out_indptr, int32_t* out_indices, void* workspace,
                 size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GUMAP_H */
