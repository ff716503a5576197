// tc_scan.cu -- dispatch of the hot scans between the tensor-core engine and
// the exact SIMT kernels.
#include <cstring>

#include "common.cuh"
#include "index.cuh"
#include "kernels.cuh"
#include "search.cuh"
#include "tc_scan.cuh"

namespace rbc {

// 0 = auto, 1 = exact SIMT only, 2 = the filtered engines (tensor cores, else the fp32 SIMT
// filter) wherever supported, 3 = the fp32 SIMT filter for every brute-force-shaped scan
// (tests: the L2 SIMT path)
static int g_engine = 0;

bool force_exact_engine() { return g_engine == 1; }

// Brute-force-shaped scans below this many (query, point) pairs stay on the exact SIMT scan
// in auto mode: the tensor-core path's operand preparation and host round trips cost more
// than the scan (e.g. cfg1's 1k x 100 one-shot search: 0.03 ms SIMT vs 0.26 ms).
int64_t tc_min_pairs() { return g_engine == 2 ? 0 : g_engine == 3 ? INT64_MAX : (int64_t(1) << 24); }
// ... and the fp32 SIMT filter pays from a few million pairs (its grouping and launch
// sequence cost ~20 us)
int64_t simt_min_pairs() { return g_engine >= 2 ? 0 : (int64_t(1) << 22); }

static unsigned __float_as_uint_host(float f) {
    unsigned u;
    std::memcpy(&u, &f, sizeof(u));
    return u;
}

__global__ void maxabs_kernel(const float *__restrict__ a, int64_t count, unsigned *__restrict__ out) {
    unsigned m = 0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        m = max(m, __float_as_uint(a[i]) & 0x7FFFFFFFu);  // |a| bits; nan sorts above inf
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

bool tc_range_ok(const float *a, int64_t count, cudaStream_t st) {
    if (count <= 0) return true;
    DevBuf<unsigned> m;
    if (m.alloc(1, st) != RBC_OK) return false;
    unsigned h = 0xFFFFFFFFu;
    if (cudaMemsetAsync(m.get(), 0, sizeof(unsigned), st) != cudaSuccess) return false;
    maxabs_kernel<<<grid_for(count, 256, 148 * 16), 256, 0, st>>>(a, count, m.get());
    note_launch();
    if (cudaMemcpyAsync(&h, m.get(), sizeof(h), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return false;
    return h <= __float_as_uint_host(kTcMaxAbs);
}

int nearest_rows(const float *q, int64_t nq, const float *x, int64_t n, int d, int metric, uint64_t *keys,
                 cudaStream_t st, const float *x4) {
    if (!force_exact_engine() && tc_bf_supported(nq, n, d, metric, 1) && tc_range_ok(q, nq * d, st) &&
        tc_range_ok(x, n * d, st))
        return tc_bf_keys(q, nq, x, n, d, 1, keys, st);
    if (!force_exact_engine() && simt_supported(d, 1) && nq * n >= simt_min_pairs())
        return simt_dense_topk(q, nq, x, n, d, metric, 1, nullptr, keys, st, x4);
    AllSrc src{x, n, d};
    return launch_topk(q, nq, d, metric, 1, src, keys, st);
}

int bf_search_keys(const float *q, int64_t nq, const float *x, int64_t n, int d, int metric, int k, uint64_t *keys,
                   cudaStream_t st) {
    if (!force_exact_engine() && tc_bf_supported(nq, n, d, metric, k) && tc_range_ok(q, nq * d, st) &&
        tc_range_ok(x, n * d, st))
        return tc_bf_keys(q, nq, x, n, d, k, keys, st);
    if (!force_exact_engine() && simt_supported(d, k) && nq * n >= simt_min_pairs())
        return simt_dense_topk(q, nq, x, n, d, metric, k, nullptr, keys, st);
    if (!force_exact_engine() && select_large_supported(nq, n, d, k))
        return select_topk_large(q, nq, x, n, d, metric, k, keys, st);
    if (k > kMaxWarpK) return topk_sorted_all(q, nq, x, n, d, metric, k, keys, st);
    AllSrc src{x, n, d};
    return launch_topk(q, nq, d, metric, k, src, keys, st);
}

int stage1_distances(const rbc_index *idx, const float *q, int64_t nq, float *d1, cudaStream_t st) {
    return pairwise(q, nq, idx->reps, idx->nr, idx->d, idx->metric, d1, st);
}

int64_t stage2_work_capacity(const rbc_index *idx, int64_t nq) {
    const int64_t ntiles = (nq + 127) / 128;
    return ntiles * idx->s2_work_per_tile + 64;
}

void stage2_note_work(const rbc_index *idx, int64_t nq, int64_t needed) {
    const int64_t ntiles = (nq + 127) / 128;
    // headroom: the tile composition (and so the union sizes) varies a little from call to
    // call, and every overflow costs a stage-2 re-run plus a graph re-capture
    const int64_t avg = (needed + ntiles - 1) / (ntiles > 0 ? ntiles : 1);
    const int64_t per = avg + avg / 4 + 8;
    if (per > idx->s2_work_per_tile) idx->s2_work_per_tile = per;
}

int stage2_scan(const rbc_index *idx, const float *q, int64_t nq, int k, const PruneOut &po, uint64_t *keys,
                cudaStream_t st) {
    if (!force_exact_engine() && tc_stage2_supported(idx, k) && tc_range_ok(q, nq * idx->d, st)) {
        DevBuf<int64_t> status;
        RBC_CHECK(status.alloc(2, st));
        for (int attempt = 0; attempt < 2; ++attempt) {
            const int64_t cap = stage2_work_capacity(idx, nq);
            RBC_CHECK(tc_stage2(idx, q, nq, k, po, keys, cap, status.get(), st));
            int64_t h[2] = {0, 0};
            RBC_CUDA(cudaMemcpyAsync(h, status.get(), sizeof(h), cudaMemcpyDeviceToHost, st));
            RBC_CUDA(cudaStreamSynchronize(st));
            last_overflow_count() = h[1];
            if (h[0] <= cap) return RBC_OK;
            stage2_note_work(idx, nq, h[0]);
        }
    }
    last_overflow_count() = 0;
    if (!force_exact_engine() && simt_exact_supported(idx, nq, k))
        return simt_exact_stage2(idx, q, nq, k, po.seg_off.get(), po.nseg.get(), po.seg_list.get(), po.seg_len.get(),
                                 po.gamma.get(), po.total_segs, keys, st);
    return stage2_exact(idx, q, nq, k, po, keys, st);
}

}  // namespace rbc

extern "C" int rbc_set_engine(int mode) {
    if (mode < 0 || mode > 3)
        return rbc::fail(RBC_EINVAL, "engine must be 0 (auto), 1 (exact), 2 (filtered engines) or 3 (SIMT filter)");
    rbc::g_engine = mode;
    return RBC_OK;
}

extern "C" int64_t rbc_stage2_overflows(void) { return rbc::last_overflow_count(); }
