/*
 * etree.h -- C ABI of the B200 E-Tree / E-Forest ADC library (libetree.so).
 *
 * Hot path of "Accelerated Distance Computation with Encoding Tree for High
 * Dimensional Data" (arXiv 1509.05186).  Citations: P:n = PAPER.md line n,
 * S:n = SPEC.md line n, A<n> = reading n in DESIGN.md §3.
 *
 * Conventions (all entry points)
 * ------------------------------
 * - Every call returns et_status (ET_OK = 0).  On error a thread-local message
 *   is available from et_last_error().  Arguments are validated before any
 *   launch; no output is written on a validation error.
 * - Ownership: the CALLER owns every buffer passed in (host or device, as each
 *   argument says).  The LIBRARY owns et_index (built by et_build_*, released
 *   with et_index_free).  An index is immutable after build and may be queried
 *   concurrently from different streams provided each call gets its own
 *   workspace.
 * - Query calls are asynchronous on `stream` (a cudaStream_t passed as void*;
 *   NULL = legacy default stream) and never synchronise the host.  Build calls
 *   are synchronous (they upload the index).
 * - Layouts: vectors fp32 row-major [n][d]; codes uint8 row-major [n][M];
 *   codebooks fp32 [M][K][d/M] (S:143 order); distance tables fp32 [Q][M][K];
 *   distances are squared L2 (no sqrt).  K <= 256, d % M == 0.
 * - Ids: int32.  A database vector is addressed by its SLOT (its row in the
 *   codes array given to the build) and reported by its ID (ids[slot], or the
 *   slot itself when ids == NULL).  Top-k orders by (distance, id) ascending
 *   (A14); missing entries are (+inf, -1).
 * - Device: every device pointer must live on the current CUDA device.
 */
#ifndef ETREE_H
#define ETREE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum et_status {
  ET_OK = 0,
  ET_ERR_INSUFFICIENT_DATA = 1,   /* S:69   n < K                               */
  ET_ERR_SUBSPACE_SPLIT = 2,      /* S:69   d % M != 0                          */
  ET_ERR_INVALID_VECTOR = 3,      /* S:69   non-finite input                    */
  ET_ERR_DIMENSION = 4,           /* S:79   length mismatch                     */
  ET_ERR_INVALID_CODE = 5,        /* S:89   code byte >= K                      */
  ET_ERR_CONFIG = 6,              /* S:119  parameter mismatch / bad split / k  */
  ET_ERR_PRECONDITION = 7,        /* S:208  unsorted input etc.                 */
  ET_ERR_EMPTY = 8,               /* S:208  N == 0                              */
  ET_ERR_CORRUPT = 9,             /* S:218  malformed buffer                    */
  ET_ERR_CUDA = 10,               /* a CUDA runtime error (message has it)      */
  ET_ERR_OOM = 11,                /* device allocation failed                   */
  ET_ERR_WORKSPACE = 12           /* workspace too small                        */
} et_status;

typedef struct et_index et_index;

/* Per-tree statistics (§4.1).  For an IVF index the
 * numbers are summed over all inverted lists. */
typedef struct et_tree_stats {
  int64_t N;               /* ids stored in this tree (4N bytes)                */
  int32_t M;               /* code bytes (levels) of this tree                          */
  int32_t layer0;          /* first code byte this tree covers (forests)                */
  int64_t L1;              /* internal nodes                                            */
  int64_t L2;              /* leaves = distinct (projected) codes                       */
  int64_t total_postfix;   /* sum over leaves of M-1-depth                              */
  int64_t lookups;         /* L1 + L2 + total_postfix = table lookups per query */
  int64_t L2_records;      /* leaf records with the 7-bit n' <= 127 chaining (A9)       */
  int64_t paper_bytes;     /* 4N + 2(L1 + L2_records) + chained postfix bytes   */
  int64_t device_bytes;    /* bytes of this tree's device layout         */
  int64_t groups;          /* id groups (leaves, or forest tuples) -- index-wide        */
  int64_t scan_lookups;    /* index-wide: table lookups per query of the GPU scan before
                              pruning (E-Tree: = lookups; fused E-Forest: each tree's
                              Distance Context over the tuple sequence) */
} et_tree_stats;

const char* et_last_error(void);
const char* et_version(void);

/* ---------------------------------------------------------------------------
 * PQ training and encoding (reading A15).  Not timed.
 * ------------------------------------------------------------------------- */

/* M independent k-means (k-means++ seeding from `seed`, then `lloyd_iters`
 * Lloyd iterations; empty cluster -> farthest point; argmin ties -> lowest k).
 * train: HOST fp32 [n][d].  codebooks: HOST fp32 [M][K][d/M] (written).
 * objective_hist: optional HOST double [M][lloyd_iters] (objective after each
 * assignment step; non-increasing).  Uses the current device for the
 * assignment steps.  Errors: n < K, d % M, non-finite input, K > 256. */
et_status et_build_codebooks(const float* train, int64_t n, int32_t d, int32_t M,
                             int32_t K, int32_t lloyd_iters, uint64_t seed,
                             float* codebooks, double* objective_hist);

/* Coarse quantizer for IVF ("K'"): k-means++ seeding from `seed`
 * then `lloyd_iters` Lloyd iterations over full d-dimensional vectors.
 * train: HOST fp32 [n][d]; centroids: HOST fp32 [nlist][d] (written);
 * objective_hist: optional HOST double [lloyd_iters].  1 <= nlist <= 65536. */
et_status et_build_coarse(const float* train, int64_t n, int32_t d, int32_t nlist,
                          int32_t lloyd_iters, uint64_t seed, float* centroids,
                          double* objective_hist);

/* Encode: code byte m = argmin_k ||x_m - c_m(k)||^2, fp32 direct difference,
 * ties -> lowest k.  codebooks, x: DEVICE; codes: DEVICE uint8 [n][M].
 * centroids/assign optional (both DEVICE, may be NULL): if given, the residual
 * x - centroids[assign[i]] is encoded (IVF). */
et_status et_encode(const float* codebooks, int32_t d, int32_t M, int32_t K,
                    const float* x, int64_t n, const float* centroids,
                    const int32_t* assign, uint8_t* codes, void* stream);

/* Nearest coarse centroid per vector (IVF list assignment; ties -> lower
 * cell).  x: DEVICE [n][d]; centroids: DEVICE [nlist][d]; assign: DEVICE int32. */
et_status et_assign(const float* centroids, int32_t nlist, int32_t d,
                    const float* x, int64_t n, int32_t* assign, void* stream);

/* ---------------------------------------------------------------------------
 * Index build (Algorithm 1 semantics P:157-180, path compression P:153-154,
 * chunked concatenation P:217-218).  Synchronous; inputs are HOST memory.
 * ------------------------------------------------------------------------- */

/* One E-Tree over all M bytes (M <= 8 on the GPU; deeper codes use a forest).
 * codes: HOST uint8 [n][M].  ids: HOST int32 [n] or NULL (ids = slots).
 * byte_perm: HOST int32 [M] or NULL (chunk order P:358-371; identity). */
et_status et_build_etree(const uint8_t* codes, const int32_t* ids, int64_t n,
                         int32_t M, int32_t K, const int32_t* byte_perm,
                         et_index** out);

/* E-Forest: T trees over the contiguous byte ranges split[t]..split[t+1]-1
 * (A13); split: HOST int32 [T+1], split[0]=0, split[T]=M, each
 * range 1..8 bytes.  T = 1 is the E-Tree. */
et_status et_build_eforest(const uint8_t* codes, const int32_t* ids, int64_t n,
                           int32_t M, int32_t K, const int32_t* byte_perm,
                           int32_t T, const int32_t* split, et_index** out);

/* Flat (uncompressed) layout of the same codes: one leaf per slot, LCP 0, so
 * the scan performs naive ADC's N*M lookups (the comparison of P:376-377 on
 * the same kernel).  M <= 8. */
et_status et_build_flat(const uint8_t* codes, const int32_t* ids, int64_t n,
                        int32_t M, int32_t K, et_index** out);

/* IVF index: one E-Tree per inverted list.  codes: residual codes
 * HOST [n][M]; list_of: HOST int32 [n] list of each vector (0..nlist-1);
 * coarse: HOST fp32 [nlist][d] (uploaded; used for residual tables);
 * codebooks: HOST fp32 [M][K][d/M] residual codebook (uploaded).
 * Errors: ET_ERR_INVALID_VECTOR for a non-finite centroid or codeword. */
et_status et_build_ivf(const uint8_t* codes, const int32_t* ids, int64_t n,
                       int32_t M, int32_t K, const int32_t* list_of,
                       int32_t nlist, const float* coarse, int32_t d,
                       const float* codebooks, et_index** out);

et_status et_index_stats(const et_index* index, int32_t tree, et_tree_stats* out);
/* Host-only: run the E-Tree/E-Forest build of et_build_eforest without a GPU
 * and return the T per-tree statistics (out: HOST et_tree_stats [T]). */
et_status et_build_stats(const uint8_t* codes, const int32_t* ids, int64_t n,
                         int32_t M, int32_t K, const int32_t* byte_perm,
                         int32_t T, const int32_t* split, et_tree_stats* out);
/* trees in the index (T), groups, N, M, K */
et_status et_index_info(const et_index* index, int32_t* T, int64_t* n,
                        int32_t* M, int32_t* K, int64_t* groups, int32_t* nlist);
void      et_index_free(et_index* index);

/* ---------------------------------------------------------------------------
 * Query path (the timed hot path).  All DEVICE pointers, async on `stream`.
 * ------------------------------------------------------------------------- */

/* Distance tables: luts[q][m][k] = sum_j (x_q[m*s+j] - C[m][k][j])^2
 * in fp32, direct difference, j ascending (no GEMM expansion: DESIGN.md §5). */
et_status et_compute_luts(const float* codebooks, int32_t d, int32_t M, int32_t K,
                          const float* queries, int64_t Q, float* luts, void* stream);

/* Bytes of device workspace et_etree_distances / et_etree_topk need. */
et_status et_workspace_size(const et_index* index, int64_t Q, int32_t k,
                            int32_t nprobe, size_t* bytes);

/* Inner-product tables (maximum inner product search; "extend ADC
 * to ... scalar product"; reading A26): luts[q][m][k] =
 * B[q][m] - <q_m, c_m(k)> with B[q][m] = max_k <q_m, c_m(k)> (fp32, the dot
 * product as a j-ascending FMA chain), offsets[q] = sum_m B[q][m].  Every entry
 * is >= 0, so et_etree_topk(luts = these) returns the k largest inner products
 * <q, x_hat> = offsets[q] - dist.  codebooks [M][K][d/M], queries [Q][d],
 * luts [Q][M][K], offsets [Q]: DEVICE fp32.  Errors: as et_compute_luts. */
et_status et_compute_ip_luts(const float* codebooks, int32_t d, int32_t M, int32_t K,
                             const float* queries, int64_t Q, float* luts, float* offsets,
                             void* stream);

/* The launch plan et_etree_topk (k > 0) or et_etree_distances (k <= 0) uses
 * for Q queries on the current device: query chunks (one CTA each, <= 32
 * queries), leaf segments per chunk (S) and lockstep leaf streams per scan
 * warp.  Host only (no launch).  Errors: ET_ERR_CONFIG (null argument, Q < 1,
 * IVF index: its chunks depend on the probes). */
et_status et_plan_info(const et_index* index, int64_t Q, int32_t k, int32_t* n_chunks,
                       int32_t* S, int32_t* streams);

/* Full output: out[q][slot] = ADC distance of database slot for
 * query q, [Q][n].  Either `luts` ([Q][M][K]) or `queries` ([Q][d]) + the
 * codebooks the index was built against must be given (queries => the tables
 * are computed inside the scan kernel).  Not for IVF indexes. */
et_status et_etree_distances(const et_index* index, const float* codebooks,
                             int32_t d, const float* luts, const float* queries,
                             int64_t Q, float* out, void* workspace,
                             size_t workspace_bytes, void* stream);

/* Fused top-k (north_star item 4): for each query the k smallest
 * (distance, id) pairs; dist: DEVICE fp32 [Q][k]; ids: DEVICE int32 [Q][k].
 * 1 <= k <= 256.  Tables as for et_etree_distances.  Launches:
 * a memset of the per-query thresholds, the scan kernel (fused tables +
 * Distance-Context scan + candidates; for forests the per-tree partials and
 * the tuple join), and the finalize kernel.  `workspace` (DEVICE, caller-owned,
 * et_workspace_size bytes) must not be shared by calls in flight at the same
 * time.  Errors: ET_ERR_CONFIG (null output, k out of range, IVF index, Q < 0),
 * ET_ERR_WORKSPACE (too small), ET_ERR_CUDA (launch failure). */
et_status et_etree_topk(const et_index* index, const float* codebooks, int32_t d,
                        const float* luts, const float* queries, int64_t Q,
                        int32_t k, float* dist, int32_t* ids, void* workspace,
                        size_t workspace_bytes, void* stream);

/* et_etree_topk from HOST buffers (the end-to-end call; north_star item 4's
 * top-k with the queries' upload and the results' read-back pipelined):
 * the Q queries are split into n_batches contiguous batches
 * (n_batches <= 0: et_host_batches' default, >= 16 queries per SM per batch,
 * at most 8); batch b's queries are copied host -> device on a library copy
 * stream while batch b - 1 is searched on `stream` (table build, scan and
 * finalize exactly as et_etree_topk, whose results it returns bit for bit:
 * the per-query arithmetic does not depend on the batch) and batch b - 2's
 * results are copied device -> host on a second copy stream.
 * queries_host: HOST fp32 [Q][d] (page-locked for the copies to overlap);
 * dist_host / ids_host: HOST fp32 / int32 [Q][k]; queries_dev: DEVICE fp32
 * [Q][d] staging; dist_dev / ids_dev: DEVICE [Q][k] staging (all caller-owned,
 * none may be touched until `stream` has passed the call); codebooks: DEVICE
 * (the index's, as et_etree_topk).  workspace: et_workspace_size of the
 * largest batch, ceil(Q / n_batches) queries.  Asynchronous: the host
 * outputs are complete once `stream` reaches the point after the call (the
 * call makes `stream` wait for the last copy).  The copy streams and events
 * are per host thread and device.  Errors: as et_etree_topk (checked before
 * anything is enqueued), ET_ERR_DIMENSION (d <= 0). */
et_status et_host_batches(int64_t Q, int32_t n_batches, int32_t* out);
et_status et_etree_topk_host(const et_index* index, const float* codebooks, int32_t d,
                             const float* queries_host, int64_t Q, int32_t k,
                             float* dist_host, int32_t* ids_host, int32_t n_batches,
                             float* queries_dev, float* dist_dev, int32_t* ids_dev,
                             void* workspace, size_t workspace_bytes, void* stream);

/* Leaf extra byte ("we quantized on the extra information to 1
 * Byte ... and store the extra information on the leaf node"; for Additive
 * Quantization it is Eq. 1's non-zero third term).
 * et_index_set_extra attaches one byte per database vector to a single E-Tree
 * index: extra = HOST uint8 [n], slot order of the codes given to the build,
 * n == N.  The byte lives on the leaf, so it must be a function of the code.
 * Errors: ET_ERR_CONFIG (not a single tree), ET_ERR_DIMENSION (n != N),
 * ET_ERR_INVALID_CODE (two vectors with the same code and different bytes).
 * et_etree_topk_extra is et_etree_topk with dist = (sum_m T[m][code[m]]) +
 * extra_table[e] (extra_table: DEVICE fp32 [256], entries >= 0 -- a
 * quantizer's decode table shifted to start at 0; 8-level trees).  Errors as
 * et_etree_topk, plus ET_ERR_CONFIG without extra bytes. */
et_status et_index_set_extra(et_index* index, const uint8_t* extra, int64_t n);
et_status et_etree_topk_extra(const et_index* index, const float* codebooks, int32_t d,
                              const float* luts, const float* queries, int64_t Q, int32_t k,
                              const float* extra_table, float* dist, int32_t* ids,
                              void* workspace, size_t workspace_bytes, void* stream);

/* IVF search: probe the nprobe nearest coarse cells (fp32 direct difference,
 * ties -> lower cell), residual tables per (query, cell), per-list E-Tree
 * scan, fused top-k.  probes: optional DEVICE int32 [Q][nprobe] output.
 * Queries are not checked on the host (they are device data, the call is
 * async): a non-finite query's coarse distances are treated as +inf, so its
 * probes are the lowest cell indices and its distances +inf/NaN -- defined,
 * never an out-of-bounds access. */
et_status et_ivf_topk(const et_index* index, const float* queries, int64_t Q,
                      int32_t nprobe, int32_t k, float* dist, int32_t* ids,
                      int32_t* probes, void* workspace, size_t workspace_bytes,
                      void* stream);

/* Merge G per-shard top-k lists (after an all-gather) into one:
 * in_dist/in_ids: DEVICE [G][Q][k] (as gathered); out: DEVICE [Q][k].
 * Order (distance, id); entries with id < 0 are empty. */
et_status et_merge_topk(const float* in_dist, const int32_t* in_ids, int32_t G,
                        int64_t Q, int32_t k, float* out_dist, int32_t* out_ids,
                        void* stream);

/* Multi-GPU shard plan (host only, no GPU).  P:217-218: sub-structures built
 * separately and concatenated form the whole HMS, so cutting the sorted codes
 * between first-level subtrees (first code byte) gives G independent trees
 * whose union of top-k lists is the global top-k.
 * codes: HOST [n][M]; bounds: HOST int32 [G+1] output, bounds[0] = 0,
 * bounds[G] = K; shard r holds the codes whose byte 0 is in
 * [bounds[r], bounds[r+1]); bounds[r] (0 < r < G) is the smallest byte value
 * v with G * #(byte0 < v) >= r * n (kept >= bounds[r-1]).  A shard may be
 * empty (the caller then contributes (+inf, -1) lists).
 * Errors: ET_ERR_CONFIG (null pointer, G < 1, K outside 1..256, M < 1). */
et_status et_shard_bounds(const uint8_t* codes, int64_t n, int32_t M, int32_t G,
                          int32_t K, int32_t* bounds);
/* The same cut from a first-byte histogram: hist HOST int64 [K] (e.g. summed
 * over ranks that each hold part of the codes). */
et_status et_shard_bounds_hist(const int64_t* hist, int32_t K, int32_t G, int32_t* bounds);

/* IVF shard plan (host only): whole inverted lists to G ranks by LPT --
 * lists in decreasing size (ties: lower list first), each to the currently
 * least-loaded rank (ties: lower rank).  list_sizes: HOST int64 [nlist];
 * owner: HOST int32 [nlist] output.  Errors: ET_ERR_CONFIG. */
et_status et_shard_lists(const int64_t* list_sizes, int32_t nlist, int32_t G, int32_t* owner);

/* Naive ADC on the GPU (comparison kernel): out[q][slot] =
 * sum_m luts[q][m][codes[slot][m]], m ascending.  codes DEVICE [n][M]. */
et_status et_flat_adc(const float* luts, int64_t Q, int32_t M, int32_t K,
                      const uint8_t* codes, int64_t n, float* out, void* stream);

/* Number of kernel launches issued by this process (all entry points). */
int64_t et_launch_count(void);

/* Per-kernel timing (measurement support): when enabled, every launch issued
 * by the query entry points is bracketed by CUDA events recorded on its own
 * stream.  et_timing_get synchronises on the recorded events and returns the
 * accumulated milliseconds and launch count of kernel `name` ("luts", "fill",
 * "scan", "finalize", "gather"); returns 0 if that kernel never ran. */
void et_timing_enable(int on);
void et_timing_reset(void);
int  et_timing_get(const char* name, double* total_ms, int64_t* count);

#ifdef __cplusplus
}
#endif
#endif /* ETREE_H */
