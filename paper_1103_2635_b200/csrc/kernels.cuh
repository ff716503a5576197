// kernels.cuh -- internal launcher declarations and candidate sources.
#pragma once

#include "common.cuh"

namespace rbc {

constexpr int kMaxWarpK = 64;  // largest k served by the register top-k paths

// ---- candidate sources for the exact warp scans ----------------------------
// for_each(i, lane, f) visits a lane-strided share of query i's candidates,
// calling f(row_ptr, global_id).

// all rows of x (bf_search, brute_force.py:165-186)
struct AllSrc {
    const float *x;
    int64_t n;
    int d;
    template <class F>
    __device__ __forceinline__ void for_each(int64_t, int lane, F &&f) const {
        for (int64_t j = lane; j < n; j += 32) f(x + j * d, static_cast<uint32_t>(j));
    }
};

// explicit id lists per query, CSR (bf_search_subset, brute_force.py:189-217)
struct IdSrc {
    const float *x;
    const int64_t *ids;
    const int64_t *off;
    int d;
    template <class F>
    __device__ __forceinline__ void for_each(int64_t i, int lane, F &&f) const {
        for (int64_t c = off[i] + lane; c < off[i + 1]; c += 32) {
            const int64_t id = ids[c];
            f(x + id * d, static_cast<uint32_t>(id));
        }
    }
};

// one row of a fixed-width list table chosen per query (one-shot search:
// the s-list of the nearest representative, search.py:116-120)
struct RowSrc {
    const float *x;
    const int32_t *lists;  // [n_reps, s] point ids
    const int32_t *row;    // [nq] chosen row per query
    int s;
    int d;
    template <class F>
    __device__ __forceinline__ void for_each(int64_t i, int lane, F &&f) const {
        const int32_t *l = lists + static_cast<int64_t>(row[i]) * s;
        for (int c = lane; c < s; c += 32) {
            const int32_t id = l[c];
            f(x + static_cast<int64_t>(id) * d, static_cast<uint32_t>(id));
        }
    }
};

// ranges of the list-ordered point copy (exact search stage 2,
// search.py:183-186): query i scans segments seg_off[i] .. seg_off[i]+seg_cnt[i],
// segment s = rows [start[s], start[s]+len[s]) of xp whose ids are perm[].
struct SegSrc {
    const float *xp;
    const int32_t *perm;
    const int64_t *seg_start;
    const int32_t *seg_len;
    const int64_t *seg_off;
    const int32_t *seg_cnt;
    int d;
    template <class F>
    __device__ __forceinline__ void for_each(int64_t i, int lane, F &&f) const {
        for (int64_t s = seg_off[i]; s < seg_off[i] + seg_cnt[i]; ++s) {
            const int64_t st = seg_start[s];
            const int32_t len = seg_len[s];
            for (int32_t j = lane; j < len; j += 32) f(xp + (st + j) * d, static_cast<uint32_t>(perm[st + j]));
        }
    }
};

// segments of a query subset (overflow fallback of the tensor-core scan):
// query i of the subset is qmap[i] of the segment CSR
struct SegSubSrc {
    const float *xp;
    const int32_t *perm;
    const int64_t *seg_start;
    const int32_t *seg_len;
    const int64_t *seg_off;
    const int32_t *seg_cnt;
    const int32_t *qmap;
    int d;
    template <class F>
    __device__ __forceinline__ void for_each(int64_t i, int lane, F &&f) const {
        const int64_t qi = qmap[i];
        for (int64_t s = seg_off[qi]; s < seg_off[qi] + seg_cnt[qi]; ++s) {
            const int64_t st = seg_start[s];
            const int32_t len = seg_len[s];
            for (int32_t j = lane; j < len; j += 32) f(xp + (st + j) * d, static_cast<uint32_t>(perm[st + j]));
        }
    }
};

int pairwise(const float *a, int64_t m, const float *b, int64_t p, int d, int metric, float *out, cudaStream_t st);

template <class Src>
int launch_topk(const float *q, int64_t nq, int d, int metric, int k, const Src &src, uint64_t *out,
                cudaStream_t st);

int topk_sorted_all(const float *q, int64_t nq, const float *x, int64_t n, int d, int metric, int k, uint64_t *out,
                    cudaStream_t st);

int count_within(const float *q, int64_t nq, const float *x, int64_t n, int d, int metric, const double *thr, int nt,
                 int strict, int64_t *counts, float *dmax, cudaStream_t st);

int unpack_keys(const uint64_t *keys, int64_t count, int64_t *ids, float *dists, int *n_empty, cudaStream_t st);

int merge_parts(const uint64_t *keys, int parts, int64_t nq, int k_in, int k_out, uint64_t *out, cudaStream_t st);

}  // namespace rbc
