/*
 * rbc_b200.h -- C-ABI of the B200-native Random Ball Cover hot path.
 *
 * Drop-in boundary for the reference package rbcover 0.1.0 (arXiv 1103.2635).
 * The reference's only native cut is the numba pair `_l2_block(a, b, out)` /
 * `_l1_block(a, b, out)` (metric.py:36-54) behind the Python API; every entry
 * point below replaces one reference function (cited per symbol) so that a
 * ctypes binding on the reference side can route its hot path here (see
 * INTEGRATION.md).
 *
 * Conventions
 *  - plain pointers + sizes; no torch types.  Unless a function name ends in
 *    `_host`, every array pointer is DEVICE memory and `stream` is a
 *    cudaStream_t (NULL = legacy default stream).  Calls are stream-ordered and
 *    asynchronous unless documented otherwise.
 *  - metric codes follow the RBCI file format (rbc.py:41): 0 = l2, 1 = l1.
 *  - point ids are int64 at the boundary (numpy int64 in the reference) and
 *    must be < 2^32 (the key64 packing of brute_force.py:62-68).
 *  - distances are bit-identical to the reference arithmetic
 *    (fp32 inputs, fp64 k-sequential accumulate without FMA, sqrt, one round
 *    to fp32; metric.py:36-54); ordering is ascending key64 =
 *    (f32 bits << 32) | id, i.e. nearest first, lowest id on ties.
 *  - return value: RBC_OK (0) or an error code; rbc_last_error() returns the
 *    calling thread's last message.  Argument errors map to the reference's
 *    ValueError (the Python layer validates first, as the reference does).
 */
#ifndef RBC_B200_H
#define RBC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { RBC_L2 = 0, RBC_L1 = 1 };

enum {
    RBC_OK = 0,
    RBC_EINVAL = 1,   /* bad argument (reference: ValueError)               */
    RBC_ECUDA = 2,    /* CUDA runtime / launch failure                      */
    RBC_ENOMEM = 3,   /* device allocation failed                           */
    RBC_EFEWCAND = 4  /* a query has fewer candidates than k
                         (reference: bf_search_subset ValueError,
                          brute_force.py:405-406)                            */
};

/* Per-query instrumentation of the exact search, structure-of-arrays form of
 * SearchStats (search.py:43-59).  reps_total == dists_step1 == n_reps. */
typedef struct rbc_search_stats {
    float *gamma;                /* [nq] k-th smallest rep distance          */
    int32_t *reps_pruned_radius; /* [nq] search.py:194                       */
    int32_t *reps_pruned_3gamma; /* [nq] search.py:195                       */
    int64_t *candidates;         /* [nq] candidates_examined                 */
} rbc_search_stats;

typedef struct rbc_index rbc_index; /* device-resident index (opaque) */

const char *rbc_last_error(void);
int rbc_abi_version(void);
/* Number of GPU kernels launched through the library (process-wide). */
int64_t rbc_launch_count(void);

/* Optional CUDA-event timing of the search phases on the launching stream
 * (0 = stage 1, 1 = pruning, 2 = stage 2 scan, 3 = build, 4 = bf scan).
 * enable(1) clears and starts recording; read() synchronises the events and
 * returns the summed milliseconds and the number of intervals per phase. */
int rbc_profile_enable(int on);
int rbc_profile_read(double *ms, int64_t *count, int32_t n_phases);

/* Engine selection for the heavy scans: 0 = auto (tcgen05 filter + exact
 * fp64 re-rank for L2, the fp32 SIMT filter + exact fp64 re-rank for L1 and
 * where the tensor cores do not apply, each where the scan is large enough to
 * pay; the default), 1 = exact fp64 SIMT only, 2 = the filtered engines
 * wherever supported, at any size, 3 = the fp32 SIMT filter for every
 * brute-force-shaped scan (L2 too).  All produce identical results; 1-3 exist
 * for A/B checks. */
int rbc_set_engine(int mode);
/* Queries of the last exact search whose candidate buffer overflowed and
 * were recomputed by the exact SIMT scan (diagnostic). */
int64_t rbc_stage2_overflows(void);
/* Brute-force scans (bf_search, build assignment, one-shot nearest rep, one-shot
 * list scan) served by the tcgen05 engine since the library loaded (diagnostic:
 * lets tests prove the tensor-core path ran). */
int64_t rbc_tc_bf_calls(void);
/* Launches of the tcgen05 list-scan kernel (stage2_tc_kernel: exact-search stage 2
 * and every tensor-core brute force) since the library loaded (diagnostic). */
int64_t rbc_tc_scan_calls(void);
/* Launches of the fp32 SIMT filter scan (simt_scan_kernel: the L1 engine, and small
 * L2 scans) since the library loaded (diagnostic). */
int64_t rbc_simt_scan_calls(void);
/* Large-k selections (k > 32: one-shot build s-lists, bf_search with large k) served by
 * the sampled-threshold engine, and the queries it handed to the exact full sort
 * (diagnostic). */
int64_t rbc_select_calls(void);
int64_t rbc_select_fallbacks(void);
/* Query batches of the exact search whose stage 1 + pruning ran the filtered engine
 * (filter_stage1.cu: d > 64 or L1), and the batches it handed back to the exact
 * |Q| x |R| path (diagnostic). */
int64_t rbc_filter_stage1_calls(void);
int64_t rbc_filter_stage1_fallbacks(void);

/* metric.py:57-76 pairwise_distances (and brute_force.py:220-251
 * distance_rows): out[m,p] = dist(a[i], b[j]), bit-exact. */
int rbc_pairwise_distances(const float *a, int64_t m, const float *b, int64_t p, int32_t d, int32_t metric,
                           float *out, void *stream);

/* brute_force.py:165-186 bf_search (the _scan_matrix core, :139-162): the k
 * nearest of every query over all of x, rows sorted by key64. */
int rbc_bf_search(const float *q, int64_t nq, const float *x, int64_t n, int32_t d, int32_t metric, int32_t k,
                  int64_t *ids, float *dists, void *stream);

/* bf_search over a PREPARED operand (the same results as rbc_bf_search): the
 * points are copied once into the tcgen05 scan's operand form (L2, d <= 64: a
 * partition into ~sqrt(n)/2 lists of f16 residuals; otherwise a plain copy for
 * the exact SIMT scan) so repeated searches over the same points -- the
 * reference's report.run_baseline loop (report.py:62-95) -- skip that work.
 * The handle is released with rbc_index_destroy. */
int rbc_bf_prepare(const float *x, int64_t n, int32_t d, int32_t metric, rbc_index **out, void *stream);
int rbc_bf_search_prepared(const rbc_index *bf, const float *q, int64_t nq, int32_t k, int64_t *ids, float *dists,
                           void *stream);

/* eval.py:21-27 ball_count, :117-130 rank_error, :133-164 claim1_counts, :44-107 estimate_expansion_rate and
 * report.py:72-95 rank_errors, batched: for query i and each of its n_thresholds thresholds t (row-major
 * thresholds[i * n_thresholds + t]), counts[i * n_thresholds + t] = #{ j : f64(dist(q_i, x_j)) < t } when strict,
 * <= t otherwise, with the reference's fp32 distance.  max_dist (nullable) receives max_j dist(q_i, x_j).
 * Per-query shared state is 4*d + 140*n_thresholds bytes and must fit in 46 KB. */
int rbc_count_within(const float *q, int64_t nq, const float *x, int64_t n, int32_t d, int32_t metric,
                     const double *thresholds, int32_t n_thresholds, int32_t strict, int64_t *counts, float *max_dist,
                     void *stream);

/* brute_force.py:189-217 bf_search_subset, batched: query i scans
 * x[subset_ids[subset_offsets[i] : subset_offsets[i+1]]] (duplicate-free,
 * validated by the caller); ids are global. */
int rbc_bf_search_subsets(const float *q, int64_t nq, const float *x, int64_t n, int32_t d, int32_t metric,
                          int32_t k, const int64_t *subset_ids, const int64_t *subset_offsets, int64_t *ids,
                          float *dists, void *stream);

/* brute_force.py:97-106 merge_neighbor_lists generalised to P partial lists
 * per query: keys[P][nq][k_in] key64 rows (UINT64_MAX = empty) -> the k_out
 * smallest per query, sorted.  Used for the rep-sharded multi-GPU merge. */
int rbc_merge_topk(const uint64_t *keys, int32_t parts, int64_t nq, int32_t k_in, int32_t k_out, int64_t *ids,
                   float *dists, void *stream);

/* rbc.py:57-59 _bernoulli_draw: numpy PCG64(default_rng(seed)) stream, id i
 * included iff random() < p.  (state, inc) are the 128-bit PCG64 state
 * words from numpy's bit_generator.state.  ids_out needs n slots; *count_out
 * (HOST) receives the count.  Synchronises the stream. */
int rbc_bernoulli_draw(int64_t n, double p, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                       uint64_t inc_lo, int64_t *ids_out, int64_t *count_out, void *stream);

/* rbc.py:147-180 build_exact: owner = nearest rep (lowest rep position on
 * ties), lists sorted by (dist, id), radius = last dist (0 if empty).
 * rep_ids ascending.  Outputs: list_ids[n], list_offsets[n_reps+1],
 * list_dists[n], radii[n_reps]. */
int rbc_build_exact(const float *x, int64_t n, int32_t d, int32_t metric, const int64_t *rep_ids, int64_t n_reps,
                    int64_t *list_ids, int64_t *list_offsets, float *list_dists, float *radii, void *stream);

/* rbc.py:183-200 build_one_shot: row p = the s nearest points of rep p in
 * key64 order; radii[p] = the s-th distance. */
int rbc_build_one_shot(const float *x, int64_t n, int32_t d, int32_t metric, const int64_t *rep_ids,
                       int64_t n_reps, int32_t s, int64_t *list_ids, float *radii, void *stream);

/* Device index over the outputs of the builds above (RbcExactIndex,
 * rbc.py:87-115 / RbcOneShotIndex, rbc.py:118-137).  The index copies what
 * it needs; inputs may be freed afterwards.  Synchronises the stream. */
int rbc_index_exact_create(const float *x, int64_t n, int32_t d, int32_t metric, const int64_t *rep_ids,
                           int64_t n_reps, const int64_t *list_ids, const int64_t *list_offsets,
                           const float *list_dists, const float *radii, rbc_index **out, void *stream);
int rbc_index_one_shot_create(const float *x, int64_t n, int32_t d, int32_t metric, const int64_t *rep_ids,
                              int64_t n_reps, const int64_t *list_ids, int32_t s, const float *radii,
                              rbc_index **out, void *stream);
/* Rep-sharded exact index (paper §7 future work): every
 * shard keeps all reps and radii (stage 1 and pruning are identical on
 * every shard) but only the lists with owned_mask[p] != 0 (HOST array). */
int rbc_index_exact_create_shard(const float *x, int64_t n, int32_t d, int32_t metric, const int64_t *rep_ids,
                                 int64_t n_reps, const int64_t *list_ids, const int64_t *list_offsets,
                                 const float *list_dists, const float *radii, const uint8_t *owned_mask,
                                 rbc_index **out, void *stream);
/* Sharded build: the representative shard of one rank
 * built from the entries it RECEIVED, without the full point set.  Every rank holds
 * all representatives (rows reps[n_reps,d], ids, global radii); the rank's m entries
 * are (ids[m], owner rep position[m], dist[m], rows[m,d]) in increasing id order, as the
 * all-to-all of the per-rank assignments delivers them.  The lists of the owned reps are
 * sorted by (dist, id) (rbc.py:168), the others stay empty; search with
 * rbc_exact_search_keys and merge over the ranks (rbc_merge_topk). */
int rbc_index_exact_create_local(const float *reps, const int64_t *rep_ids, int64_t n_reps, const float *radii,
                                 int64_t n_total, int32_t d, int32_t metric, const float *rows, const int64_t *ids,
                                 const int64_t *owner, const float *dist, int64_t m, rbc_index **out, void *stream);
/* radii[p] = max dist over the entries owned by p (0 if none): a rank's share of the
 * list radii (rbc.py:172-175), combined across ranks with an all-reduce(MAX). */
int rbc_local_list_radii(const int64_t *owner, const float *dist, int64_t m, int64_t n_reps, float *radii,
                         void *stream);
int rbc_index_destroy(rbc_index *idx);
/* Bytes of device memory held by the index. */
int64_t rbc_index_device_bytes(const rbc_index *idx);

/* search.py:150-208 exact_query_batch: ids/dists [nq,k]; stats may be NULL
 * members.  On a shard index, rows hold the shard-local top-k (missing
 * entries id = -1, dist = +inf) and stats count the shard's candidates. */
int rbc_exact_search(const rbc_index *idx, const float *q, int64_t nq, int32_t k, int64_t *ids, float *dists,
                     rbc_search_stats stats, void *stream);
/* Same, returning packed key64 rows [nq,k] (UINT64_MAX = empty) for merging. */
int rbc_exact_search_keys(const rbc_index *idx, const float *q, int64_t nq, int32_t k, uint64_t *keys,
                          rbc_search_stats stats, void *stream);

/* search.py:90-141 one_shot_query_batch: gamma[nq] may be NULL. */
int rbc_one_shot_search(const rbc_index *idx, const float *q, int64_t nq, int32_t k, int64_t *ids, float *dists,
                        float *gamma, void *stream);

/* End-to-end variants: q and every output in HOST memory; the call copies
 * q to the device, searches, copies the results back and synchronises. */
int rbc_exact_search_host(const rbc_index *idx, const float *q, int64_t nq, int32_t k, int64_t *ids, float *dists,
                          rbc_search_stats stats, void *stream);
int rbc_one_shot_search_host(const rbc_index *idx, const float *q, int64_t nq, int32_t k, int64_t *ids,
                             float *dists, float *gamma, void *stream);

/* search.py:217-238 range_query for one query (HOST q; outputs HOST, capacity
 * cap); returns the number of points within radius in *count (may exceed
 * cap: call again with a larger buffer). */
int rbc_range_query_host(const rbc_index *idx, const float *q, double radius, int64_t cap, int64_t *ids,
                         float *dists, int64_t *count, void *stream);

/* search.py:62-74 prune_representatives: mask[p] = survives, evaluated in
 * float64 on float64 inputs exactly as numpy does. */
int rbc_prune_representatives(const double *rep_dists, const double *radii, int64_t n_reps, double gamma,
                              uint8_t *mask, void *stream);

/* search.py:77-82 list_cutoff, batched over thresholds: out[t] = number of
 * leading entries of the ascending list that are <= thresholds[t]. */
int rbc_list_cutoff(const double *sorted, int64_t m, const double *thresholds, int64_t n_thresholds, int64_t *out,
                    void *stream);

/* Diagnostic: one 128 x n x 64 f16 tcgen05.mma tile (A [128][64], B [n][64]
 * row-major f16, device) -> c [128][n] f32, through the same UMMA
 * descriptor / TMEM path as the stage-2 engine.  n in {16, 32, ..., 256}. */
int rbc_tc_selftest(const void *a, const void *b, float *c, int32_t n, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* RBC_B200_H */
