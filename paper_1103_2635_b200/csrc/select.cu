// select.cu -- k nearest points for large k (k > 32): the one-shot build's s-lists
// (rbc.py:196-200: bf_search(reps, X, s) for every representative) and bf_search /
// the report baseline with large k (brute_force.py:165-186, report.py:62-95).
//
// Instead of materialising and sorting all n keys of every query (topk_sorted_all), the
// k smallest are selected through a threshold:
//   1. a strided sample of X (every st-th row, st = k / 8) is scanned by the SIMT filter
//      engine for each query's 32 nearest sample points; the 32nd sample distance tau is,
//      with overwhelming probability on non-adversarial data, beyond the k-th distance of
//      all of X (about 8 sample points are expected inside the k nearest);
//   2. one fp32 pass over all (query, point) pairs (rep-stationary tiles in shared
//      memory, one point per thread) counts the points with S <= thr = tau^p fac and
//      collects, with their exact key64 (reference arithmetic), every point with
//      S <= thr fac^2 -- a superset of the true k nearest whenever the count reaches k
//      (any k points with S <= thr have reference distances <= (thr fac)^(1/p), so every
//      member of the true top-k has S <= thr fac^2);
//   3. each query's collected keys are sorted (CUB segmented radix sort) and the first k
//      kept.
// A query whose count stays below k (an unrepresentative sample) or whose collection
// overflows its buffer is recomputed by the exact full sort, so the keys are always the
// reference's.
#include <cub/cub.cuh>

#include <algorithm>
#include <atomic>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "tc_scan.cuh"

namespace rbc {

namespace {

constexpr int kQT = 64;    // queries per collect tile (shared memory)
constexpr int kCT = 256;   // collect threads (one point each)
constexpr int kSampleK = 32;

__global__ void gather_strided_kernel(const float *__restrict__ x, int64_t rows, int d, int64_t stride,
                                      float *__restrict__ out) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < rows * d;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = t / d;
        out[t] = x[r * stride * d + (t - r * d)];
    }
}

// fp32 thresholds from the exact 32nd sample distance: thr = tau^p fac (+ slack), and the
// collection bound thr fac^2
__global__ void thresholds_kernel(const uint64_t *__restrict__ skeys, int64_t nq, int d, int metric,
                                  float *__restrict__ thr) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= nq) return;
    const uint64_t key = skeys[i * kSampleK + kSampleK - 1];
    const float fac = 1.0f + static_cast<float>(4 * d + 16) * (1.0f / 16777216.0f);
    const float absl = static_cast<float>(d) * 1e-35f;
    float lo = __int_as_float(0x7f800000), hi = lo;
    if (key != kEmptyKey) {
        const float tau = key_dist(key);
        const float tp = metric == RBC_L2 ? tau * tau * (1.0f + 1.0f / 8388608.0f) : tau;
        lo = fmaf(tp, fac, absl);
        hi = fmaf(lo, fac * fac, absl);
    }
    thr[2 * i] = lo;
    thr[2 * i + 1] = hi;
}

template <int METRIC>
__device__ __forceinline__ float term32(float a, float b, float acc) {
    const float t = a - b;
    return METRIC == RBC_L2 ? fmaf(t, t, acc) : acc + fabsf(t);
}

// grid (point blocks, query tiles): thread = one point (registers), queries of the tile
// from shared memory; counts S <= thr_lo and collects exact keys of S <= thr_hi
template <int METRIC, int DMAX>
__global__ void __launch_bounds__(kCT) collect_kernel(const float *__restrict__ q, int64_t nq, const float *__restrict__ x,
                                                      int64_t n, int d, const float *__restrict__ thr, int cap,
                                                      int32_t *__restrict__ cnt_lo, int32_t *__restrict__ cnt_hi,
                                                      uint64_t *__restrict__ cand) {
    __shared__ __align__(16) float qs[kQT][DMAX];
    __shared__ float th[kQT][2];
    const int64_t q0 = static_cast<int64_t>(blockIdx.y) * kQT;
    const int qn = static_cast<int>(min(static_cast<int64_t>(kQT), nq - q0));
    for (int e = threadIdx.x; e < kQT * DMAX; e += kCT) {
        const int r = e / DMAX, c = e - r * DMAX;
        qs[r][c] = (r < qn && c < d) ? q[(q0 + r) * d + c] : 0.f;
    }
    for (int e = threadIdx.x; e < kQT * 2; e += kCT) th[e >> 1][e & 1] = (e >> 1) < qn ? thr[2 * q0 + e] : -1.f;
    __syncthreads();
    const int64_t j = static_cast<int64_t>(blockIdx.x) * kCT + threadIdx.x;
    if (j >= n) return;
    float xv[DMAX];
#pragma unroll
    for (int c = 0; c < DMAX; ++c) xv[c] = c < d ? __ldg(x + j * d + c) : 0.f;
    for (int r = 0; r < qn; ++r) {
        float a0 = 0.f, a1 = 0.f;
#pragma unroll
        for (int c = 0; c < DMAX; c += 4) {
            if (c < d) {
                const float4 qq = *reinterpret_cast<const float4 *>(&qs[r][c]);
                a0 = term32<METRIC>(qq.x, xv[c], a0);
                a1 = term32<METRIC>(qq.y, xv[c + 1], a1);
                a0 = term32<METRIC>(qq.z, xv[c + 2], a0);
                a1 = term32<METRIC>(qq.w, xv[c + 3], a1);
            }
        }
        const float S = a0 + a1;
        if (S <= th[r][1]) {
            const int64_t qi = q0 + r;
            if (S <= th[r][0]) atomicAdd(&cnt_lo[qi], 1);
            const int pos = atomicAdd(&cnt_hi[qi], 1);
            if (pos < cap) cand[qi * cap + pos] = pack_key(exact_dist<METRIC>(q + qi * d, x + j * d, d), static_cast<uint32_t>(j));
        }
    }
}

__global__ void seg_bounds_kernel(const int32_t *__restrict__ cnt_hi, int64_t nq, int cap, int *__restrict__ beg,
                                  int *__restrict__ end) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= nq) return;
    beg[i] = static_cast<int>(i * cap);
    end[i] = static_cast<int>(i * cap + min(cnt_hi[i], cap));
}

__global__ void take_first_kernel(const uint64_t *__restrict__ sorted, int64_t nq, int cap, int k,
                                  uint64_t *__restrict__ out) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t < nq * k) out[t] = sorted[(t / k) * cap + t % k];
}

__global__ void gather_rows_idx_kernel(const float *__restrict__ src, const int32_t *__restrict__ ids, int64_t rows,
                                       int d, float *__restrict__ dst) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t < rows * d) dst[t] = src[static_cast<int64_t>(ids[t / d]) * d + t % d];
}

__global__ void scatter_keys_kernel(const uint64_t *__restrict__ src, const int32_t *__restrict__ ids, int64_t rows,
                                    int k, uint64_t *__restrict__ dst) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t < rows * k) dst[static_cast<int64_t>(ids[t / k]) * k + t % k] = src[t];
}

template <int METRIC>
int launch_collect(const float *q, int64_t nq, const float *x, int64_t n, int d, const float *thr, int cap,
                   int32_t *lo, int32_t *hi, uint64_t *cand, cudaStream_t st) {
    const dim3 grid(grid_for(n, kCT), static_cast<unsigned>((nq + kQT - 1) / kQT));
    if (d <= 24) collect_kernel<METRIC, 24><<<grid, kCT, 0, st>>>(q, nq, x, n, d, thr, cap, lo, hi, cand);
    else if (d <= 64) collect_kernel<METRIC, 64><<<grid, kCT, 0, st>>>(q, nq, x, n, d, thr, cap, lo, hi, cand);
    else collect_kernel<METRIC, 128><<<grid, kCT, 0, st>>>(q, nq, x, n, d, thr, cap, lo, hi, cand);
    RBC_LAUNCHED();
    return RBC_OK;
}

std::atomic<int64_t> g_select_calls{0}, g_select_fallbacks{0};

}  // namespace

bool select_large_supported(int64_t nq, int64_t n, int d, int k) {
    const int64_t stride = std::max(1, k / 8);
    return k > kSampleK && d <= 128 && n / stride >= 2 * kSampleK && n < (int64_t(1) << 31) && nq > 0 &&
           nq * n >= simt_min_pairs();
}

int select_topk_large(const float *q, int64_t nq, const float *x, int64_t n, int d, int metric, int k, uint64_t *keys,
                      cudaStream_t st) {
    if (!select_large_supported(nq, n, d, k)) return topk_sorted_all(q, nq, x, n, d, metric, k, keys, st);
    g_select_calls.fetch_add(1);
    const int64_t stride = std::max(1, k / 8), ns = n / stride;
    // per-query candidate buffer: ~32 stride points expected below thr; the rest is headroom
    const int cap = static_cast<int>(std::min<int64_t>(n, 64 * stride + 4096));
    DevBuf<float> xs, thr;
    DevBuf<uint64_t> skeys;
    RBC_CHECK(xs.alloc(ns * d, st));
    gather_strided_kernel<<<grid_for(ns * d, 256, 148 * 64), 256, 0, st>>>(x, ns, d, stride, xs.get());
    RBC_LAUNCHED();
    RBC_CHECK(skeys.alloc(nq * kSampleK, st));
    RBC_CHECK(simt_dense_topk(q, nq, xs.get(), ns, d, metric, kSampleK, nullptr, skeys.get(), st));
    RBC_CHECK(thr.alloc(2 * nq, st));
    thresholds_kernel<<<grid_for(nq, 256), 256, 0, st>>>(skeys.get(), nq, d, metric, thr.get());
    RBC_LAUNCHED();
    // query batches bounded to ~1 GiB of candidate keys
    const int64_t qb = std::max<int64_t>(1, std::min<int64_t>(nq, (int64_t(1) << 27) / cap));
    DevBuf<int32_t> lo, hi;
    DevBuf<uint64_t> cand, sorted;
    DevBuf<int> beg, end;
    RBC_CHECK(lo.alloc(nq, st));
    RBC_CHECK(hi.alloc(nq, st));
    RBC_CHECK(cand.alloc(qb * cap, st));
    RBC_CHECK(sorted.alloc(qb * cap, st));
    RBC_CHECK(beg.alloc(qb, st));
    RBC_CHECK(end.alloc(qb, st));
    RBC_CUDA(cudaMemsetAsync(lo.get(), 0, sizeof(int32_t) * nq, st));
    RBC_CUDA(cudaMemsetAsync(hi.get(), 0, sizeof(int32_t) * nq, st));
    size_t tb = 0;
    cub::DeviceSegmentedRadixSort::SortKeys(nullptr, tb, cand.get(), sorted.get(), qb * cap, static_cast<int>(qb),
                                            beg.get(), end.get(), 0, 64, st);
    DevBuf<unsigned char> tmp;
    RBC_CHECK(tmp.alloc(tb, st));
    for (int64_t q0 = 0; q0 < nq; q0 += qb) {
        const int64_t rows = std::min(qb, nq - q0);
        if (metric == RBC_L2)
            RBC_CHECK(launch_collect<RBC_L2>(q + q0 * d, rows, x, n, d, thr.get() + 2 * q0, cap, lo.get() + q0,
                                             hi.get() + q0, cand.get(), st));
        else
            RBC_CHECK(launch_collect<RBC_L1>(q + q0 * d, rows, x, n, d, thr.get() + 2 * q0, cap, lo.get() + q0,
                                             hi.get() + q0, cand.get(), st));
        seg_bounds_kernel<<<grid_for(rows, 256), 256, 0, st>>>(hi.get() + q0, rows, cap, beg.get(), end.get());
        RBC_LAUNCHED();
        size_t tb2 = tb;
        RBC_CUDA(cub::DeviceSegmentedRadixSort::SortKeys(tmp.get(), tb2, cand.get(), sorted.get(), rows * cap,
                                                         static_cast<int>(rows), beg.get(), end.get(), 0, 64, st));
        note_launch();
        take_first_kernel<<<grid_for(rows * k, 256), 256, 0, st>>>(sorted.get(), rows, cap, k, keys + q0 * k);
        RBC_LAUNCHED();
    }
    // queries whose threshold missed (count below k, or a collection past the buffer): exact sort
    std::vector<int32_t> hlo(nq), hhi(nq);
    RBC_CUDA(cudaMemcpyAsync(hlo.data(), lo.get(), sizeof(int32_t) * nq, cudaMemcpyDeviceToHost, st));
    RBC_CUDA(cudaMemcpyAsync(hhi.data(), hi.get(), sizeof(int32_t) * nq, cudaMemcpyDeviceToHost, st));
    RBC_CUDA(cudaStreamSynchronize(st));
    std::vector<int32_t> redo;
    for (int64_t i = 0; i < nq; ++i)
        if (hlo[i] < k || hhi[i] > cap) redo.push_back(static_cast<int32_t>(i));
    if (redo.empty()) return RBC_OK;
    g_select_fallbacks.fetch_add(static_cast<int64_t>(redo.size()));
    const int64_t m = static_cast<int64_t>(redo.size());
    DevBuf<int32_t> ids;
    DevBuf<float> qr;
    DevBuf<uint64_t> kr;
    RBC_CHECK(ids.alloc(m, st));
    RBC_CHECK(qr.alloc(m * d, st));
    RBC_CHECK(kr.alloc(m * k, st));
    RBC_CUDA(cudaMemcpyAsync(ids.get(), redo.data(), sizeof(int32_t) * m, cudaMemcpyHostToDevice, st));
    gather_rows_idx_kernel<<<grid_for(m * d, 256), 256, 0, st>>>(q, ids.get(), m, d, qr.get());
    RBC_LAUNCHED();
    RBC_CHECK(topk_sorted_all(qr.get(), m, x, n, d, metric, k, kr.get(), st));
    scatter_keys_kernel<<<grid_for(m * k, 256), 256, 0, st>>>(kr.get(), ids.get(), m, k, keys);
    RBC_LAUNCHED();
    RBC_CUDA(cudaStreamSynchronize(st));
    return RBC_OK;
}

}  // namespace rbc

extern "C" int64_t rbc_select_calls(void) { return rbc::g_select_calls.load(); }
extern "C" int64_t rbc_select_fallbacks(void) { return rbc::g_select_fallbacks.load(); }
