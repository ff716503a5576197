// tc_scan.cu -- dispatch of the hot scans.
#include "common.cuh"
#include "index.cuh"
#include "kernels.cuh"
#include "search.cuh"
#include "tc_scan.cuh"

namespace rbc {

int nearest_rows(const float *q, int64_t nq, const float *x, int64_t n, int d, int metric, uint64_t *keys,
                 cudaStream_t st) {
    AllSrc src{x, n, d};
    return launch_topk(q, nq, d, metric, 1, src, keys, st);
}

int bf_search_keys(const float *q, int64_t nq, const float *x, int64_t n, int d, int metric, int k, uint64_t *keys,
                   cudaStream_t st) {
    if (k > kMaxWarpK) return topk_sorted_all(q, nq, x, n, d, metric, k, keys, st);
    AllSrc src{x, n, d};
    return launch_topk(q, nq, d, metric, k, src, keys, st);
}

int stage1_distances(const rbc_index *idx, const float *q, int64_t nq, float *d1, cudaStream_t st) {
    return pairwise(q, nq, idx->reps, idx->nr, idx->d, idx->metric, d1, st);
}

int stage2_scan(const rbc_index *idx, const float *q, int64_t nq, int k, const PruneOut &po, uint64_t *keys,
                cudaStream_t st) {
    return stage2_exact(idx, q, nq, k, po, keys, st);
}

int tc_index_prepare(rbc_index *, cudaStream_t) { return RBC_OK; }
void tc_index_release(rbc_index *) {}

}  // namespace rbc
