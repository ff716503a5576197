/*
 * rbc_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference algorithm (rbcover 0.1.0, the
 * Random Ball Cover package of arXiv 1103.2635) used as the parity checker
 * for the B200 path.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library; the product
 * path (paper_1103_2635_b200) never links or calls it.
 *
 * Pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py imports /root/reference/pkg/src/rbcover in
 * the build container and writes the tests/golden npz files); see
 * tests/test_oracle_golden.py.
 *
 * Every function cites the reference file:line it restates.  Arithmetic
 * contract (reference metric.py:36-54): fp32 inputs widened to fp64,
 * k-sequential accumulation with a separate multiply and add (compile with
 * -ffp-contract=off; no -ffast-math), sqrt in fp64, one rounding to fp32.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_L2 0
#define ORC_L1 1

/* ---- metric.py:36-44 (_l2_block) / :47-54 (_l1_block) ------------------ */
static inline float orc_dist(const float *a, const float *b, int d, int metric) {
    double acc = 0.0;
    if (metric == ORC_L2) {
        for (int k = 0; k < d; ++k) {
            double diff = (double)a[k] - (double)b[k];
            acc += diff * diff;
        }
        return (float)sqrt(acc);
    }
    for (int k = 0; k < d; ++k) acc += fabs((double)a[k] - (double)b[k]);
    return (float)acc;
}

static inline uint32_t f32_bits(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    return u;
}
static inline float bits_f32(uint32_t u) {
    float f;
    memcpy(&f, &u, 4);
    return f;
}

/* brute_force.py:62-68 (_pack_keys): (f32 bits << 32) | id */
static inline uint64_t pack_key(float dist, uint64_t id) {
    return ((uint64_t)f32_bits(dist) << 32) | (id & 0xFFFFFFFFull);
}

int orc_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* metric.py:57-76 (pairwise_distances) */
void orc_pairwise(const float *a, int64_t m, const float *b, int64_t p, int d, int metric, float *out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < p; ++j) out[i * p + j] = orc_dist(a + i * d, b + j * d, d, metric);
}

/* ---- bounded max-heap of u64 keys: the k smallest keys of a stream ------ */
static void heap_sift_down(uint64_t *h, int n, int i) {
    for (;;) {
        int l = 2 * i + 1, r = l + 1, m = i;
        if (l < n && h[l] > h[m]) m = l;
        if (r < n && h[r] > h[m]) m = r;
        if (m == i) return;
        uint64_t t = h[i];
        h[i] = h[m];
        h[m] = t;
        i = m;
    }
}
static void heap_push_bounded(uint64_t *h, int *cnt, int k, uint64_t key) {
    if (*cnt < k) {
        int i = (*cnt)++;
        h[i] = key;
        while (i > 0) {
            int p = (i - 1) / 2;
            if (h[p] >= h[i]) break;
            uint64_t t = h[p];
            h[p] = h[i];
            h[i] = t;
            i = p;
        }
    } else if (key < h[0]) {
        h[0] = key;
        heap_sift_down(h, k, 0);
    }
}
static int cmp_u64(const void *x, const void *y) {
    uint64_t a = *(const uint64_t *)x, b = *(const uint64_t *)y;
    return a < b ? -1 : (a > b ? 1 : 0);
}
static void unpack_sorted(uint64_t *h, int cnt, int64_t *ids, float *dists) {
    qsort(h, (size_t)cnt, sizeof(uint64_t), cmp_u64);
    for (int i = 0; i < cnt; ++i) {
        ids[i] = (int64_t)(h[i] & 0xFFFFFFFFull);
        dists[i] = bits_f32((uint32_t)(h[i] >> 32));
    }
}

/* brute_force.py:139-186 (_scan_matrix / bf_search): per query the k smallest
 * key64 over all of X, sorted ascending.  Tiling/threads cannot change the
 * result (key64 is a total order), so the restatement scans linearly. */
void orc_bf_topk(const float *q, int64_t nq, const float *x, int64_t n, int d, int metric, int k, int64_t *ids,
                 float *dists) {
#pragma omp parallel
    {
        uint64_t *h = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)k);
#pragma omp for schedule(dynamic, 4)
        for (int64_t i = 0; i < nq; ++i) {
            int cnt = 0;
            const float *qi = q + i * d;
            for (int64_t j = 0; j < n; ++j) heap_push_bounded(h, &cnt, k, pack_key(orc_dist(qi, x + j * d, d, metric), (uint64_t)j));
            unpack_sorted(h, cnt, ids + i * k, dists + i * k);
        }
        free(h);
    }
}

/* brute_force.py:189-217 (bf_search_subset), batched: query i scans
 * X[cand[off[i]:off[i+1]]]; global ids are reported. */
void orc_bf_subsets(const float *q, int64_t nq, const float *x, int d, int metric, int k, const int64_t *cand,
                    const int64_t *off, int64_t *ids, float *dists) {
#pragma omp parallel
    {
        uint64_t *h = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)k);
#pragma omp for schedule(dynamic, 4)
        for (int64_t i = 0; i < nq; ++i) {
            int cnt = 0;
            for (int64_t c = off[i]; c < off[i + 1]; ++c)
                heap_push_bounded(h, &cnt, k, pack_key(orc_dist(q + i * d, x + cand[c] * d, d, metric), (uint64_t)cand[c]));
            unpack_sorted(h, cnt, ids + i * k, dists + i * k);
        }
        free(h);
    }
}

/* ---- rbc.py:57-59 (_bernoulli_draw): numpy PCG64 stream ----------------
 * numpy's pcg64 step: state = state * MULT + inc, then XSL-RR output;
 * random() = (next_uint64 >> 11) * 2^-53.  Draw i is included iff
 * random() < p; ids ascending (np.flatnonzero). */
typedef unsigned __int128 u128;
#define PCG_MULT ((((u128)0x2360ED051FC65DA4ull) << 64) | (u128)0x4385DF649FCCF645ull)

static inline uint64_t xsl_rr(u128 s) {
    uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
    uint64_t v = hi ^ lo;
    unsigned rot = (unsigned)(hi >> 58);
    return (v >> rot) | (v << ((64u - rot) & 63u));
}

int64_t orc_bernoulli(int64_t n, double p, uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo,
                      int64_t *ids_out) {
    u128 s = ((u128)st_hi << 64) | st_lo;
    u128 inc = ((u128)inc_hi << 64) | inc_lo;
    int64_t cnt = 0;
    for (int64_t i = 0; i < n; ++i) {
        s = s * PCG_MULT + inc;
        double u = (double)(xsl_rr(s) >> 11) * (1.0 / 9007199254740992.0);
        if (u < p) ids_out[cnt++] = i;
    }
    return cnt;
}

/* ---- rbc.py:147-180 (build_exact) --------------------------------------
 * owner = k=1 scan of X against X[R] (lowest rep position on ties), then
 * lexsort((id, dist, owner)) into CSR lists; radius = last list dist. */
typedef struct {
    int64_t owner;
    float dist;
    int64_t id;
} orc_entry;
static int cmp_entry(const void *x, const void *y) {
    const orc_entry *a = (const orc_entry *)x, *b = (const orc_entry *)y;
    if (a->owner != b->owner) return a->owner < b->owner ? -1 : 1;
    if (a->dist != b->dist) return a->dist < b->dist ? -1 : 1;
    return a->id < b->id ? -1 : (a->id > b->id);
}

void orc_build_exact(const float *x, int64_t n, int d, int metric, const int64_t *rep_ids, int64_t nr,
                     int64_t *list_ids, int64_t *offsets, float *list_dists, float *radii) {
    orc_entry *e = (orc_entry *)malloc(sizeof(orc_entry) * (size_t)n);
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < n; ++i) {
        uint64_t best = UINT64_MAX;
        for (int64_t p = 0; p < nr; ++p) {
            uint64_t key = pack_key(orc_dist(x + i * d, x + rep_ids[p] * d, d, metric), (uint64_t)p);
            if (key < best) best = key;
        }
        e[i].owner = (int64_t)(best & 0xFFFFFFFFull);
        e[i].dist = bits_f32((uint32_t)(best >> 32));
        e[i].id = i;
    }
    qsort(e, (size_t)n, sizeof(orc_entry), cmp_entry);
    for (int64_t p = 0; p <= nr; ++p) offsets[p] = 0;
    for (int64_t i = 0; i < n; ++i) {
        list_ids[i] = e[i].id;
        list_dists[i] = e[i].dist;
        offsets[e[i].owner + 1]++;
    }
    for (int64_t p = 0; p < nr; ++p) offsets[p + 1] += offsets[p];
    for (int64_t p = 0; p < nr; ++p) radii[p] = offsets[p + 1] > offsets[p] ? list_dists[offsets[p + 1] - 1] : 0.0f;
    free(e);
}

/* rbc.py:183-200 (build_one_shot): row p = the s nearest points to rep p. */
void orc_build_one_shot(const float *x, int64_t n, int d, int metric, const int64_t *rep_ids, int64_t nr, int s,
                        int64_t *list_ids, float *radii) {
    float *dd = (float *)malloc(sizeof(float) * (size_t)(nr * s));
    float *rp = (float *)malloc(sizeof(float) * (size_t)(nr * d) + 4);
    for (int64_t p = 0; p < nr; ++p) memcpy(rp + p * d, x + rep_ids[p] * d, sizeof(float) * (size_t)d);
    orc_bf_topk(rp, nr, x, n, d, metric, s, list_ids, dd);
    for (int64_t p = 0; p < nr; ++p) radii[p] = dd[p * s + s - 1];
    free(dd);
    free(rp);
}

/* search.py:62-74 (prune_representatives), f64 comparisons. */
static inline int orc_survives(float dist, float radius, double g) {
    double d = (double)dist, r = (double)radius;
    return (d <= 3.0 * g) && ((d < g + r) || (d <= g));
}

/* search.py:77-82 (list_cutoff): #entries <= thr (f64 compare), binary search. */
int64_t orc_list_cutoff(const float *sorted, int64_t m, double thr) {
    int64_t lo = 0, hi = m;
    while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if ((double)sorted[mid] <= thr) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

static int cmp_f32(const void *x, const void *y) {
    float a = *(const float *)x, b = *(const float *)y;
    return a < b ? -1 : (a > b ? 1 : 0);
}

/* search.py:150-208 (exact_query_batch).  Stats per query: gamma,
 * reps_pruned_radius, reps_pruned_3gamma, candidates_examined
 * (reps_total = dists_step1 = nr).  Returns 0, or -(i+1) if query i has
 * fewer candidates than k (the reference raises ValueError there). */
int64_t orc_exact_query(const float *x, int d, int metric, const int64_t *rep_ids, int64_t nr,
                        const int64_t *list_ids, const int64_t *offsets, const float *list_dists,
                        const float *radii, const float *q, int64_t nq, int k, int64_t *ids, float *dists,
                        float *gamma_out, int64_t *pr_out, int64_t *p3_out, int64_t *cand_out) {
    int64_t bad = 0;
#pragma omp parallel
    {
        float *row = (float *)malloc(sizeof(float) * (size_t)nr);
        float *tmp = (float *)malloc(sizeof(float) * (size_t)nr);
        uint64_t *h = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)k);
#pragma omp for schedule(dynamic, 8)
        for (int64_t i = 0; i < nq; ++i) {
            const float *qi = q + i * d;
            for (int64_t p = 0; p < nr; ++p) row[p] = orc_dist(qi, x + rep_ids[p] * d, d, metric);
            /* search.py:181: gamma_k = k-th smallest rep distance */
            float gk;
            if (k == 1) {
                gk = row[0];
                for (int64_t p = 1; p < nr; ++p)
                    if (row[p] < gk) gk = row[p];
            } else {
                memcpy(tmp, row, sizeof(float) * (size_t)nr);
                qsort(tmp, (size_t)nr, sizeof(float), cmp_f32);
                gk = tmp[k - 1];
            }
            double g = (double)gk, cut = 4.0 * g;
            int cnt = 0;
            int64_t ncand = 0, pr = 0, p3 = 0;
            for (int64_t p = 0; p < nr; ++p) {
                double dp = (double)row[p];
                if (dp >= g + (double)radii[p] && dp > g) pr++; /* search.py:194 */
                if (dp > 3.0 * g) p3++;                        /* search.py:195 */
                if (!orc_survives(row[p], radii[p], g)) continue;
                int64_t len = orc_list_cutoff(list_dists + offsets[p], offsets[p + 1] - offsets[p], cut);
                for (int64_t c = 0; c < len; ++c) {
                    int64_t id = list_ids[offsets[p] + c];
                    heap_push_bounded(h, &cnt, k, pack_key(orc_dist(qi, x + id * d, d, metric), (uint64_t)id));
                }
                ncand += len;
            }
            if (ncand < k) {
#pragma omp critical
                bad = -(i + 1);
            }
            unpack_sorted(h, cnt, ids + i * k, dists + i * k);
            gamma_out[i] = gk;
            pr_out[i] = pr;
            p3_out[i] = p3;
            cand_out[i] = ncand;
        }
        free(row);
        free(tmp);
        free(h);
    }
    return bad;
}

/* search.py:90-141 (one_shot_query_batch): nearest rep by key64 argmin,
 * then the k smallest keys over its s-list.  gamma = d(q, r_best). */
void orc_one_shot_query(const float *x, int d, int metric, const int64_t *rep_ids, int64_t nr,
                        const int64_t *list_ids, int s, const float *q, int64_t nq, int k, int64_t *ids,
                        float *dists, float *gamma_out) {
#pragma omp parallel
    {
        uint64_t *h = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)k);
#pragma omp for schedule(dynamic, 8)
        for (int64_t i = 0; i < nq; ++i) {
            const float *qi = q + i * d;
            uint64_t best = UINT64_MAX;
            for (int64_t p = 0; p < nr; ++p) {
                uint64_t key = pack_key(orc_dist(qi, x + rep_ids[p] * d, d, metric), (uint64_t)p);
                if (key < best) best = key;
            }
            int64_t bp = (int64_t)(best & 0xFFFFFFFFull);
            int cnt = 0;
            for (int c = 0; c < s; ++c) {
                int64_t id = list_ids[bp * s + c];
                heap_push_bounded(h, &cnt, k, pack_key(orc_dist(qi, x + id * d, d, metric), (uint64_t)id));
            }
            unpack_sorted(h, cnt, ids + i * k, dists + i * k);
            gamma_out[i] = bits_f32((uint32_t)(best >> 32));
        }
        free(h);
    }
}

/* search.py:217-238 (range_query) for one query: writes up to cap ids/dists
 * sorted by (dist, id); returns the total count (may exceed cap). */
int64_t orc_range_query(const float *x, int d, int metric, const int64_t *rep_ids, int64_t nr,
                        const int64_t *list_ids, const int64_t *offsets, const float *list_dists,
                        const float *radii, const float *q, double eps, int64_t cap, int64_t *ids, float *dists) {
    uint64_t *keys = NULL;
    int64_t cnt = 0, capk = 0;
    for (int64_t p = 0; p < nr; ++p) {
        double rd = (double)orc_dist(q, x + rep_ids[p] * d, d, metric);
        if (!(rd <= eps + (double)radii[p])) continue;
        int64_t len = orc_list_cutoff(list_dists + offsets[p], offsets[p + 1] - offsets[p], eps + rd);
        for (int64_t c = 0; c < len; ++c) {
            int64_t id = list_ids[offsets[p] + c];
            float dd = orc_dist(q, x + id * d, d, metric);
            if ((double)dd <= eps) {
                if (cnt == capk) {
                    capk = capk ? 2 * capk : 64;
                    keys = (uint64_t *)realloc(keys, sizeof(uint64_t) * (size_t)capk);
                }
                keys[cnt++] = pack_key(dd, (uint64_t)id);
            }
        }
    }
    if (cnt) qsort(keys, (size_t)cnt, sizeof(uint64_t), cmp_u64);
    for (int64_t i = 0; i < cnt && i < cap; ++i) {
        ids[i] = (int64_t)(keys[i] & 0xFFFFFFFFull);
        dists[i] = bits_f32((uint32_t)(keys[i] >> 32));
    }
    free(keys);
    return cnt;
}
