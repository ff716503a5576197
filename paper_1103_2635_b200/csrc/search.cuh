// search.cuh -- internal interfaces of the search pipeline.
#pragma once

#include "common.cuh"
#include "index.cuh"

namespace rbc {

struct CastI64 {
    __host__ __device__ __forceinline__ int64_t operator()(const int32_t &v) const { return v; }
};

// Output of stage 1 + pruning for a query chunk.
struct PruneOut {
    DevBuf<float> gamma;       // [nq] gamma_k
    DevBuf<int32_t> nseg;      // [nq] non-empty surviving segments
    DevBuf<int64_t> cand;      // [nq] candidates_examined
    DevBuf<int64_t> seg_off;   // [nq+1] first segment of query i (its segments: seg_off[i] .. +nseg[i])
    DevBuf<int64_t> seg_start; // [total] first list-order position
    DevBuf<int32_t> seg_len;   // [total] cutoff length
    DevBuf<int32_t> seg_list;  // [total] rep position of the segment
    DevBuf<float> seg_d1;      // [total] exact dist(q, r_p) of the segment's list
    DevBuf<uint64_t> order_key; // [nq] (first surviving list << 24) | nearest rep: query grouping key
    DevBuf<int32_t> qorder;     // [nq] stage-1 query order (by nearest pilot), fused path only
    DevBuf<unsigned long long> s2_total;  // stage-2 work counter, zeroed by the fused stage 1 (pilot scatter)
    mutable bool s2_total_zeroed = false;  // true until the first tc_stage2 call takes it
    const float *d1 = nullptr; // stage-1 distances [nq, nr] (owned by the caller)
    int64_t total_segs = 0;
    int32_t *pr = nullptr;     // optional stats outputs (caller memory)
    int32_t *p3 = nullptr;
};

int prune(const rbc_index *idx, const float *d1, int64_t nq, int k, PruneOut &out, cudaStream_t st);
int exact_search_keys(const rbc_index *idx, const float *q, int64_t nq, int k, uint64_t *keys,
                      const rbc_search_stats &stats, cudaStream_t st);
int stage2_exact(const rbc_index *idx, const float *q, int64_t nq, int k, const PruneOut &po, uint64_t *keys,
                 cudaStream_t st);
int one_shot_search_keys(const rbc_index *idx, const float *q, int64_t nq, int k, uint64_t *keys, float *gamma,
                         cudaStream_t st);

}  // namespace rbc
