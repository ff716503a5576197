// range.cu -- epsilon-range query on the exact index (search.py:217-238).
//
// A list is scanned when dist(q, r) <= eps + psi_r (non-strict, f64), and
// only its prefix with member distance <= eps + dist(q, r); members within
// eps are appended as key64 and sorted, giving (dist, id) order.
#include <cub/cub.cuh>

#include "common.cuh"
#include "index.cuh"
#include "kernels.cuh"

namespace rbc {

template <int METRIC>
__global__ void range_scan_kernel(const float *__restrict__ q, const float *__restrict__ d1, double eps,
                                  const float *__restrict__ radii, const int64_t *__restrict__ offsets,
                                  const float *__restrict__ list_dists, const float *__restrict__ xp,
                                  const int32_t *__restrict__ perm, int d, uint64_t *__restrict__ keys,
                                  unsigned long long *__restrict__ count) {
    extern __shared__ float qs[];
    const int64_t p = blockIdx.x;
    const double rd = d1[p];
    if (!(rd <= __dadd_rn(eps, static_cast<double>(radii[p])))) return;
    for (int c = threadIdx.x; c < d; c += blockDim.x) qs[c] = q[c];
    __syncthreads();
    const float *l = list_dists + offsets[p];
    const double thr = __dadd_rn(eps, rd);
    int64_t lo = 0, hi = offsets[p + 1] - offsets[p];
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (static_cast<double>(l[mid]) <= thr) lo = mid + 1;
        else hi = mid;
    }
    for (int64_t j = threadIdx.x; j < lo; j += blockDim.x) {
        const int64_t pos = offsets[p] + j;
        const float dist = exact_dist<METRIC>(qs, xp + pos * d, d);
        if (static_cast<double>(dist) <= eps) {
            const unsigned long long slot = atomicAdd(count, 1ull);
            keys[slot] = pack_key(dist, static_cast<uint32_t>(perm[pos]));
        }
    }
}

int range_query_host(const rbc_index *idx, const float *q_host, double eps, int64_t cap, int64_t *ids, float *dists,
                     int64_t *count_out, cudaStream_t st) {
    const int d = idx->d;
    DevBuf<float> q, d1;
    DevBuf<uint64_t> keys, sorted;
    DevBuf<unsigned long long> count;
    RBC_CHECK(q.alloc(d, st));
    RBC_CHECK(d1.alloc(idx->nr, st));
    RBC_CHECK(keys.alloc(idx->n_local, st));
    RBC_CHECK(count.alloc(1, st));
    RBC_CUDA(cudaMemcpyAsync(q.get(), q_host, sizeof(float) * d, cudaMemcpyHostToDevice, st));
    RBC_CUDA(cudaMemsetAsync(count.get(), 0, sizeof(unsigned long long), st));
    RBC_CHECK(pairwise(q.get(), 1, idx->reps, idx->nr, d, idx->metric, d1.get(), st));
    const size_t smem = sizeof(float) * d;
    if (idx->metric == RBC_L2)
        range_scan_kernel<RBC_L2><<<static_cast<unsigned>(idx->nr), 128, smem, st>>>(
            q.get(), d1.get(), eps, idx->radii, idx->offsets, idx->list_dists, idx->xp, idx->perm, d, keys.get(), count.get());
    else
        range_scan_kernel<RBC_L1><<<static_cast<unsigned>(idx->nr), 128, smem, st>>>(
            q.get(), d1.get(), eps, idx->radii, idx->offsets, idx->list_dists, idx->xp, idx->perm, d, keys.get(), count.get());
    RBC_LAUNCHED();
    unsigned long long total = 0;
    RBC_CUDA(cudaMemcpyAsync(&total, count.get(), sizeof(total), cudaMemcpyDeviceToHost, st));
    RBC_CUDA(cudaStreamSynchronize(st));
    *count_out = static_cast<int64_t>(total);
    if (total == 0) return RBC_OK;
    RBC_CHECK(sorted.alloc(total, st));
    size_t tb = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tb, keys.get(), sorted.get(), static_cast<int64_t>(total), 0, 64, st);
    DevBuf<unsigned char> tmp;
    RBC_CHECK(tmp.alloc(tb, st));
    RBC_CUDA(cub::DeviceRadixSort::SortKeys(tmp.get(), tb, keys.get(), sorted.get(), static_cast<int64_t>(total), 0, 64, st));
    note_launch();
    const int64_t take = static_cast<int64_t>(total) < cap ? static_cast<int64_t>(total) : cap;
    if (take > 0) {
        DevBuf<int64_t> did;
        DevBuf<float> ddist;
        RBC_CHECK(did.alloc(take, st));
        RBC_CHECK(ddist.alloc(take, st));
        RBC_CHECK(unpack_keys(sorted.get(), take, did.get(), ddist.get(), nullptr, st));
        RBC_CUDA(cudaMemcpyAsync(ids, did.get(), sizeof(int64_t) * take, cudaMemcpyDeviceToHost, st));
        RBC_CUDA(cudaMemcpyAsync(dists, ddist.get(), sizeof(float) * take, cudaMemcpyDeviceToHost, st));
    }
    RBC_CUDA(cudaStreamSynchronize(st));
    return RBC_OK;
}

}  // namespace rbc

extern "C" int rbc_range_query_host(const rbc_index *idx, const float *q, double radius, int64_t cap, int64_t *ids,
                                    float *dists, int64_t *count, void *stream) {
    if (!idx || idx->kind != 0) return rbc::fail(RBC_EINVAL, "not an exact index");
    if (!(radius >= 0)) return rbc::fail(RBC_EINVAL, "radius must be >= 0");
    return rbc::range_query_host(idx, q, radius, cap, ids, dists, count, reinterpret_cast<cudaStream_t>(stream));
}
