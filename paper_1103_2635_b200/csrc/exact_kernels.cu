// exact_kernels.cu -- bit-exact distance blocks and exact top-k scans.
//
// These kernels evaluate the reference arithmetic (metric.py:36-54) directly
// in fp64 on the SIMT pipes.  They serve the small/irregular calls of the
// API (pairwise_distances, bf_search_subset, the one-shot list scan), the
// large-k path of bf_search/build_one_shot, and the overflow fallback of the
// tensor-core filtered scans (tc_scan.cu).  Results are independent of the
// work decomposition because selection is on unique key64 values
// (brute_force.py:8-12).
#include <algorithm>

#include <cub/cub.cuh>

#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace rbc {

// ---- pairwise distance block (metric.py:57-76) -----------------------------
// 64x64 output tile per 256-thread block, 4x4 outputs per thread, operands
// staged through shared memory 32 coordinates at a time.  Each output keeps
// its own fp64 accumulator advanced in coordinate order 0..d-1.
template <int METRIC>
__global__ void __launch_bounds__(256) pairwise_kernel(const float *__restrict__ a, int64_t m,
                                                       const float *__restrict__ b, int64_t p, int d,
                                                       float *__restrict__ out) {
    __shared__ float as[64][33];
    __shared__ float bs[64][33];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t i0 = static_cast<int64_t>(blockIdx.y) * 64, j0 = static_cast<int64_t>(blockIdx.x) * 64;
    double acc[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
    for (int k0 = 0; k0 < d; k0 += 32) {
        const int kc = min(32, d - k0);
        for (int t = threadIdx.x; t < 64 * 32; t += 256) {
            const int r = t >> 5, c = t & 31;
            as[r][c] = (i0 + r < m && c < kc) ? a[(i0 + r) * d + k0 + c] : 0.f;
            bs[r][c] = (j0 + r < p && c < kc) ? b[(j0 + r) * d + k0 + c] : 0.f;
        }
        __syncthreads();
        for (int c = 0; c < kc; ++c) {
            float av[4], bv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) av[u] = as[ty + 16 * u][c];
#pragma unroll
            for (int v = 0; v < 4; ++v) bv[v] = bs[tx + 16 * v][c];
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v)
                    acc[u][v] = __dadd_rn(acc[u][v], METRIC == RBC_L2 ? l2_term(av[u], bv[v]) : l1_term(av[u], bv[v]));
        }
        __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int64_t i = i0 + ty + 16 * u, j = j0 + tx + 16 * v;
            if (i < m && j < p)
                out[i * p + j] = METRIC == RBC_L2 ? __double2float_rn(__dsqrt_rn(acc[u][v])) : __double2float_rn(acc[u][v]);
        }
}

int pairwise(const float *a, int64_t m, const float *b, int64_t p, int d, int metric, float *out, cudaStream_t st) {
    if (m == 0 || p == 0) return RBC_OK;
    dim3 grid(grid_for(p, 64, 1 << 30), grid_for(m, 64, 65535));
    if (grid.y > 65535) return fail(RBC_EINVAL, "pairwise: too many rows for one call");
    if (metric == RBC_L2) pairwise_kernel<RBC_L2><<<grid, 256, 0, st>>>(a, m, b, p, d, out);
    else pairwise_kernel<RBC_L1><<<grid, 256, 0, st>>>(a, m, b, p, d, out);
    RBC_LAUNCHED();
    return RBC_OK;
}

// ---- warp-per-query exact top-k scans --------------------------------------
// Each lane keeps an ascending register array of its KT best key64 values
// over a strided share of the candidates, then the warp merges the 32 sorted
// arrays (warp_merge_sorted).  KT >= k, so the merge sees at least the k
// smallest keys.
constexpr int kWarpsPerBlock = 8;

template <int METRIC, int KT, class Src>
__global__ void __launch_bounds__(kWarpsPerBlock * 32) topk_warp_kernel(const float *__restrict__ q, int64_t nq,
                                                                        int d, int k, Src src,
                                                                        uint64_t *__restrict__ out) {
    extern __shared__ float qs_all[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * kWarpsPerBlock + w;
    if (i >= nq) return;
    float *qs = qs_all + w * d;
    for (int c = lane; c < d; c += 32) qs[c] = q[i * d + c];
    __syncwarp();
    uint64_t best[KT];
#pragma unroll
    for (int j = 0; j < KT; ++j) best[j] = kEmptyKey;
    src.for_each(i, lane, [&](const float *__restrict__ row, uint32_t id) {
        const uint64_t key = pack_key(exact_dist<METRIC>(qs, row, d), id);
        if (key < best[KT - 1]) sorted_insert<KT>(best, key);
    });
    warp_merge_sorted<KT>(best, k, out + i * k);
}

template <class Src, int KT>
static int launch_topk_kt(const float *q, int64_t nq, int d, int metric, int k, const Src &src, uint64_t *out,
                          cudaStream_t st) {
    const unsigned grid = grid_for(nq, kWarpsPerBlock);
    const size_t smem = sizeof(float) * kWarpsPerBlock * d;
    if (smem > 48 * 1024) return fail(RBC_EINVAL, "dimension too large for the exact scan kernel");
    if (metric == RBC_L2) topk_warp_kernel<RBC_L2, KT, Src><<<grid, kWarpsPerBlock * 32, smem, st>>>(q, nq, d, k, src, out);
    else topk_warp_kernel<RBC_L1, KT, Src><<<grid, kWarpsPerBlock * 32, smem, st>>>(q, nq, d, k, src, out);
    RBC_LAUNCHED();
    return RBC_OK;
}

// ---- k > 64: every candidate key of a query batch, segmented radix sort ------------------
// The reference accepts any k <= |R| (exact, search.py:167-170) or k <= s (one-shot,
// search.py:104-105).  Above the register top-k width the candidates' exact keys are
// materialised per query (batches of <= 2^27 keys), sorted per query with CUB, and the
// first k kept (missing entries = empty keys when a query has fewer than k candidates).
template <class Src>
__global__ void __launch_bounds__(kWarpsPerBlock * 32) count_cand_kernel(int64_t nq, Src src, int64_t *__restrict__ cnt) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * kWarpsPerBlock + w;
    if (i >= nq) return;
    int64_t c = 0;
    src.for_each(i, lane, [&](const float *, uint32_t) { ++c; });
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) cnt[i] = c;
}

template <int METRIC, class Src>
__global__ void __launch_bounds__(kWarpsPerBlock * 32) cand_keys_kernel(const float *__restrict__ q, int64_t q0,
                                                                        int64_t rows, int d, Src src,
                                                                        const int64_t *__restrict__ off,
                                                                        uint64_t *__restrict__ keys) {
    extern __shared__ float qs_all[];
    __shared__ unsigned long long pos[kWarpsPerBlock];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t r = static_cast<int64_t>(blockIdx.x) * kWarpsPerBlock + w;
    if (r >= rows) return;
    const int64_t i = q0 + r;
    float *qs = qs_all + w * d;
    for (int c = lane; c < d; c += 32) qs[c] = q[i * d + c];
    if (lane == 0) pos[w] = 0;
    __syncwarp();
    uint64_t *dst = keys + (off[i] - off[q0]);
    src.for_each(i, lane, [&](const float *__restrict__ row, uint32_t id) {
        const unsigned long long p = atomicAdd(&pos[w], 1ull);
        dst[p] = pack_key(exact_dist<METRIC>(qs, row, d), id);
    });
}

__global__ void rebase_offsets_kernel(const int64_t *__restrict__ off, int64_t q0, int64_t rows,
                                      int64_t *__restrict__ out) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t <= rows) out[t] = off[q0 + t] - off[q0];
}

__global__ void take_k_kernel(const uint64_t *__restrict__ sorted, const int64_t *__restrict__ off, int64_t q0,
                              int64_t rows, int k, uint64_t *__restrict__ out) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t >= rows * k) return;
    const int64_t r = t / k, j = t % k;
    const int64_t a = off[q0 + r] - off[q0], n = off[q0 + r + 1] - off[q0 + r];
    out[(q0 + r) * k + j] = j < n ? sorted[a + j] : kEmptyKey;
}

template <class Src>
static int topk_large(const float *q, int64_t nq, int d, int metric, int k, const Src &src, uint64_t *out,
                      cudaStream_t st) {
    const size_t qsmem = sizeof(float) * kWarpsPerBlock * d;
    if (qsmem > 48 * 1024) return fail(RBC_EINVAL, "dimension too large for the exact scan kernel");
    DevBuf<int64_t> cnt, off;
    RBC_CHECK(cnt.alloc(nq, st));
    RBC_CHECK(off.alloc(nq + 1, st));
    count_cand_kernel<Src><<<grid_for(nq, kWarpsPerBlock), kWarpsPerBlock * 32, 0, st>>>(nq, src, cnt.get());
    RBC_LAUNCHED();
    RBC_CUDA(cudaMemsetAsync(off.get(), 0, sizeof(int64_t), st));
    size_t tb = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tb, cnt.get(), off.get() + 1, nq, st);
    {
        DevBuf<unsigned char> tmp;
        RBC_CHECK(tmp.alloc(tb, st));
        RBC_CUDA(cub::DeviceScan::InclusiveSum(tmp.get(), tb, cnt.get(), off.get() + 1, nq, st));
    }
    std::vector<int64_t> h(nq + 1);
    RBC_CUDA(cudaMemcpyAsync(h.data(), off.get(), sizeof(int64_t) * (nq + 1), cudaMemcpyDeviceToHost, st));
    RBC_CUDA(cudaStreamSynchronize(st));
    const int64_t budget = int64_t(1) << 27;  // keys per batch (1 GiB of key64)
    int64_t maxb = 0;
    for (int64_t q0 = 0; q0 < nq;) {  // largest batch, for the buffer sizes
        int64_t q1 = q0 + 1;
        while (q1 < nq && q1 - q0 < 65535 && h[q1 + 1] - h[q0] <= budget) ++q1;
        maxb = h[q1] - h[q0] > maxb ? h[q1] - h[q0] : maxb;
        q0 = q1;
    }
    DevBuf<uint64_t> keys, sorted;
    DevBuf<int64_t> boff;
    RBC_CHECK(keys.alloc(maxb, st));
    RBC_CHECK(sorted.alloc(maxb, st));
    RBC_CHECK(boff.alloc(65536, st));
    for (int64_t q0 = 0; q0 < nq;) {
        int64_t q1 = q0 + 1;
        while (q1 < nq && q1 - q0 < 65535 && h[q1 + 1] - h[q0] <= budget) ++q1;
        const int64_t rows = q1 - q0, total = h[q1] - h[q0];
        if (metric == RBC_L2)
            cand_keys_kernel<RBC_L2, Src><<<grid_for(rows, kWarpsPerBlock), kWarpsPerBlock * 32, qsmem, st>>>(
                q, q0, rows, d, src, off.get(), keys.get());
        else
            cand_keys_kernel<RBC_L1, Src><<<grid_for(rows, kWarpsPerBlock), kWarpsPerBlock * 32, qsmem, st>>>(
                q, q0, rows, d, src, off.get(), keys.get());
        RBC_LAUNCHED();
        rebase_offsets_kernel<<<grid_for(rows + 1, 256), 256, 0, st>>>(off.get(), q0, rows, boff.get());
        RBC_LAUNCHED();
        size_t sb = 0;
        cub::DeviceSegmentedRadixSort::SortKeys(nullptr, sb, keys.get(), sorted.get(), total, static_cast<int>(rows),
                                                boff.get(), boff.get() + 1, 0, 64, st);
        DevBuf<unsigned char> tmp;
        RBC_CHECK(tmp.alloc(sb, st));
        RBC_CUDA(cub::DeviceSegmentedRadixSort::SortKeys(tmp.get(), sb, keys.get(), sorted.get(), total,
                                                         static_cast<int>(rows), boff.get(), boff.get() + 1, 0, 64,
                                                         st));
        note_launch();
        take_k_kernel<<<grid_for(rows * k, 256), 256, 0, st>>>(sorted.get(), off.get(), q0, rows, k, out);
        RBC_LAUNCHED();
        q0 = q1;
    }
    return RBC_OK;
}

template <class Src>
int launch_topk(const float *q, int64_t nq, int d, int metric, int k, const Src &src, uint64_t *out,
                cudaStream_t st) {
    if (nq == 0) return RBC_OK;
    if (k <= 1) return launch_topk_kt<Src, 1>(q, nq, d, metric, k, src, out, st);
    if (k <= 4) return launch_topk_kt<Src, 4>(q, nq, d, metric, k, src, out, st);
    if (k <= 16) return launch_topk_kt<Src, 16>(q, nq, d, metric, k, src, out, st);
    if (k <= kMaxWarpK) return launch_topk_kt<Src, kMaxWarpK>(q, nq, d, metric, k, src, out, st);
    return topk_large(q, nq, d, metric, k, src, out, st);
}

template int launch_topk<AllSrc>(const float *, int64_t, int, int, int, const AllSrc &, uint64_t *, cudaStream_t);
template int launch_topk<IdSrc>(const float *, int64_t, int, int, int, const IdSrc &, uint64_t *, cudaStream_t);
template int launch_topk<SegSrc>(const float *, int64_t, int, int, int, const SegSrc &, uint64_t *, cudaStream_t);
template int launch_topk<RowSrc>(const float *, int64_t, int, int, int, const RowSrc &, uint64_t *, cudaStream_t);
template int launch_topk<SegSubSrc>(const float *, int64_t, int, int, int, const SegSubSrc &, uint64_t *, cudaStream_t);

// ---- key64 rows -> (ids, dists) -------------------------------------------
__global__ void unpack_keys_kernel(const uint64_t *__restrict__ keys, int64_t count, int64_t *__restrict__ ids,
                                   float *__restrict__ dists, int *__restrict__ n_empty) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < count;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint64_t key = keys[t];
        unpack_to(key, ids + t, dists + t);
        if (key == kEmptyKey && n_empty) atomicAdd(n_empty, 1);
    }
}

// ---- ball counts (eval.py:21-27 ball_count, :117-130 rank_error, :133-164 claim1_counts, :44-107
// estimate_expansion_rate; report.py:72-95 rank_errors) ---------------------------------------------------------
// Warp per query over all of x.  Every distance is the reference's fp32 value (exact_dist); query i counts, for
// each of its nt thresholds, the points with f64(dist) < thr (strict) or <= thr (closed) -- numpy's comparison of
// an fp32 row against a double.  Each lane keeps private counters in shared memory (stride 33: the final
// column sums are conflict-free), so no n-length distance row is ever written.  Optional: the row maximum.
template <int METRIC>
__global__ void __launch_bounds__(256) count_within_kernel(const float *__restrict__ q, int64_t nq,
                                                           const float *__restrict__ x, int64_t n, int d,
                                                           const double *__restrict__ thr, int nt, int strict,
                                                           int64_t *__restrict__ counts, float *__restrict__ dmax) {
    extern __shared__ __align__(16) unsigned char cw_smem[];
    const int nw = blockDim.x >> 5, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * nw + w;
    if (i >= nq) return;
    const size_t q_bytes = (static_cast<size_t>(nw) * d * sizeof(float) + 15) & ~size_t(15);
    float *qs = reinterpret_cast<float *>(cw_smem) + static_cast<size_t>(w) * d;
    double *ts = reinterpret_cast<double *>(cw_smem + q_bytes) + static_cast<size_t>(w) * nt;
    uint32_t *cs = reinterpret_cast<uint32_t *>(cw_smem + q_bytes + static_cast<size_t>(nw) * nt * sizeof(double)) +
                   static_cast<size_t>(w) * nt * 33;
    for (int c = lane; c < d; c += 32) qs[c] = q[i * d + c];
    for (int t = lane; t < nt; t += 32) ts[t] = thr[i * nt + t];
    for (int t = 0; t < nt; ++t) cs[t * 33 + lane] = 0;
    __syncwarp();
    float mx = 0.f;
    for (int64_t j = lane; j < n; j += 32) {
        const float dv = exact_dist<METRIC>(qs, x + j * d, d);
        mx = fmaxf(mx, dv);
        const double dd = dv;
        if (strict) {
            for (int t = 0; t < nt; ++t) cs[t * 33 + lane] += dd < ts[t] ? 1u : 0u;
        } else {
            for (int t = 0; t < nt; ++t) cs[t * 33 + lane] += dd <= ts[t] ? 1u : 0u;
        }
    }
    __syncwarp();
    for (int t = lane; t < nt; t += 32) {
        int64_t sum = 0;
        for (int l = 0; l < 32; ++l) sum += cs[t * 33 + l];
        counts[i * nt + t] = sum;
    }
    // distances are >= 0, so their bit patterns order like unsigned integers
    const uint32_t m = __reduce_max_sync(0xffffffffu, __float_as_uint(mx));
    if (dmax != nullptr && lane == 0) dmax[i] = __uint_as_float(m);
}

int count_within(const float *q, int64_t nq, const float *x, int64_t n, int d, int metric, const double *thr, int nt,
                 int strict, int64_t *counts, float *dmax, cudaStream_t st) {
    if (nq == 0) return RBC_OK;
    const size_t per_warp = static_cast<size_t>(d) * sizeof(float) + static_cast<size_t>(nt) * (sizeof(double) + 33 * 4);
    constexpr size_t kBudget = 46 * 1024;
    if (per_warp + 16 > kBudget) return fail(RBC_EINVAL, "count_within: too many thresholds per query for this d");
    const int nw = static_cast<int>(std::min<size_t>(8, (kBudget - 16) / per_warp));
    const size_t smem = ((static_cast<size_t>(nw) * d * sizeof(float) + 15) & ~size_t(15)) +
                        static_cast<size_t>(nw) * nt * (sizeof(double) + 33 * 4);
    const int64_t blocks = (nq + nw - 1) / nw;
    if (blocks > 0x7FFFFFFF) return fail(RBC_EINVAL, "count_within: too many queries for one call");
    if (metric == RBC_L2)
        count_within_kernel<RBC_L2><<<static_cast<unsigned>(blocks), nw * 32, smem, st>>>(q, nq, x, n, d, thr, nt, strict,
                                                                                         counts, dmax);
    else
        count_within_kernel<RBC_L1><<<static_cast<unsigned>(blocks), nw * 32, smem, st>>>(q, nq, x, n, d, thr, nt, strict,
                                                                                         counts, dmax);
    RBC_LAUNCHED();
    return RBC_OK;
}

int unpack_keys(const uint64_t *keys, int64_t count, int64_t *ids, float *dists, int *n_empty, cudaStream_t st) {
    if (count == 0) return RBC_OK;
    unpack_keys_kernel<<<grid_for(count, 256, 148 * 32), 256, 0, st>>>(keys, count, ids, dists, n_empty);
    RBC_LAUNCHED();
    return RBC_OK;
}

// ---- P-way merge of partial key rows (multi-GPU rep-shard merge) -----------
// keys[part][i][c], c < k_in  ->  the k_out smallest per query i.
template <int KT>
__global__ void merge_parts_kernel(const uint64_t *__restrict__ keys, int parts, int64_t nq, int k_in, int k_out,
                                   uint64_t *__restrict__ out) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * kWarpsPerBlock + w;
    if (i >= nq) return;
    uint64_t best[KT];
#pragma unroll
    for (int j = 0; j < KT; ++j) best[j] = kEmptyKey;
    for (int t = lane; t < parts * k_in; t += 32) {
        const int part = t / k_in, c = t % k_in;
        const uint64_t key = keys[(static_cast<int64_t>(part) * nq + i) * k_in + c];
        if (key < best[KT - 1]) sorted_insert<KT>(best, key);
    }
    warp_merge_sorted<KT>(best, k_out, out + i * k_out);
}

__global__ void gather_parts_kernel(const uint64_t *__restrict__ keys, int parts, int64_t nq, int k_in,
                                    uint64_t *__restrict__ flat) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int64_t w = static_cast<int64_t>(parts) * k_in;
    if (t >= nq * w) return;
    const int64_t i = t / w, r = t % w;
    flat[t] = keys[((r / k_in) * nq + i) * k_in + r % k_in];
}

__global__ void take_prefix_kernel(const uint64_t *__restrict__ sorted, int64_t rows, int64_t n, int k,
                                   uint64_t *__restrict__ out);
__global__ void seg_offsets_kernel(int64_t *off, int64_t rows, int64_t n);

int merge_parts(const uint64_t *keys, int parts, int64_t nq, int k_in, int k_out, uint64_t *out, cudaStream_t st) {
    if (nq == 0) return RBC_OK;
    const unsigned grid = grid_for(nq, kWarpsPerBlock);
    if (k_out <= 1) merge_parts_kernel<1><<<grid, kWarpsPerBlock * 32, 0, st>>>(keys, parts, nq, k_in, k_out, out);
    else if (k_out <= 4) merge_parts_kernel<4><<<grid, kWarpsPerBlock * 32, 0, st>>>(keys, parts, nq, k_in, k_out, out);
    else if (k_out <= 16) merge_parts_kernel<16><<<grid, kWarpsPerBlock * 32, 0, st>>>(keys, parts, nq, k_in, k_out, out);
    else if (k_out <= kMaxWarpK)
        merge_parts_kernel<kMaxWarpK><<<grid, kWarpsPerBlock * 32, 0, st>>>(keys, parts, nq, k_in, k_out, out);
    else {
        // large k: flatten each query's parts, segmented radix sort, keep the prefix
        const int64_t w = static_cast<int64_t>(parts) * k_in;
        DevBuf<uint64_t> flat, sorted;
        DevBuf<int64_t> off;
        RBC_CHECK(flat.alloc(nq * w, st));
        RBC_CHECK(sorted.alloc(nq * w, st));
        RBC_CHECK(off.alloc(nq + 1, st));
        gather_parts_kernel<<<grid_for(nq * w, 256), 256, 0, st>>>(keys, parts, nq, k_in, flat.get());
        RBC_LAUNCHED();
        seg_offsets_kernel<<<grid_for(nq + 1, 256), 256, 0, st>>>(off.get(), nq, w);
        RBC_LAUNCHED();
        size_t tb = 0;
        cub::DeviceSegmentedRadixSort::SortKeys(nullptr, tb, flat.get(), sorted.get(), nq * w, nq, off.get(),
                                                off.get() + 1, 0, 64, st);
        DevBuf<unsigned char> tmp;
        RBC_CHECK(tmp.alloc(tb, st));
        RBC_CUDA(cub::DeviceSegmentedRadixSort::SortKeys(tmp.get(), tb, flat.get(), sorted.get(), nq * w, nq,
                                                         off.get(), off.get() + 1, 0, 64, st));
        note_launch();
        take_prefix_kernel<<<grid_for(nq * k_out, 256), 256, 0, st>>>(sorted.get(), nq, w, k_out, out);
    }
    RBC_LAUNCHED();
    return RBC_OK;
}

// ---- large-k path: all keys of a query chunk, segmented radix sort ---------
// Used for k > kMaxWarpK (the one-shot build's s-lists, the report's
// k=512 baseline).  Keys of `chunk` rows are materialised, sorted per row
// with CUB, and the first k of each row kept.
template <int METRIC>
__global__ void all_keys_kernel(const float *__restrict__ q, int64_t rows, const float *__restrict__ x, int64_t n,
                                int d, uint64_t *__restrict__ keys) {
    extern __shared__ float qs[];
    const int64_t r = blockIdx.y;
    for (int c = threadIdx.x; c < d; c += blockDim.x) qs[c] = q[r * d + c];
    __syncthreads();
    for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < n;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x)
        keys[r * n + j] = pack_key(exact_dist<METRIC>(qs, x + j * d, d), static_cast<uint32_t>(j));
}

__global__ void seg_offsets_kernel(int64_t *off, int64_t rows, int64_t n) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t <= rows) off[t] = t * n;
}

__global__ void take_prefix_kernel(const uint64_t *__restrict__ sorted, int64_t rows, int64_t n, int k,
                                   uint64_t *__restrict__ out) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t < rows * k) out[t] = sorted[(t / k) * n + t % k];
}

int topk_sorted_all(const float *q, int64_t nq, const float *x, int64_t n, int d, int metric, int k,
                    uint64_t *out, cudaStream_t st) {
    if (nq == 0) return RBC_OK;
    const int64_t budget = int64_t(1) << 27;  // keys per chunk (1 GiB of key64)
    int64_t chunk = budget / n;
    if (chunk < 1) chunk = 1;
    if (chunk > nq) chunk = nq;
    if (chunk > 65535) chunk = 65535;
    DevBuf<uint64_t> keys, sorted;
    DevBuf<int64_t> off;
    RBC_CHECK(keys.alloc(chunk * n, st));
    RBC_CHECK(sorted.alloc(chunk * n, st));
    RBC_CHECK(off.alloc(chunk + 1, st));
    size_t tmp_bytes = 0;
    cub::DeviceSegmentedRadixSort::SortKeys(nullptr, tmp_bytes, keys.get(), sorted.get(), chunk * n, chunk, off.get(),
                                            off.get() + 1, 0, 64, st);
    DevBuf<unsigned char> tmp;
    RBC_CHECK(tmp.alloc(tmp_bytes, st));
    for (int64_t r0 = 0; r0 < nq; r0 += chunk) {
        const int64_t rows = nq - r0 < chunk ? nq - r0 : chunk;
        dim3 grid(grid_for(n, 256, 64), static_cast<unsigned>(rows));
        const size_t smem = sizeof(float) * d;
        if (metric == RBC_L2) all_keys_kernel<RBC_L2><<<grid, 256, smem, st>>>(q + r0 * d, rows, x, n, d, keys.get());
        else all_keys_kernel<RBC_L1><<<grid, 256, smem, st>>>(q + r0 * d, rows, x, n, d, keys.get());
        RBC_LAUNCHED();
        seg_offsets_kernel<<<grid_for(rows + 1, 256), 256, 0, st>>>(off.get(), rows, n);
        RBC_LAUNCHED();
        size_t tb = tmp_bytes;
        RBC_CUDA(cub::DeviceSegmentedRadixSort::SortKeys(tmp.get(), tb, keys.get(), sorted.get(), rows * n,
                                                         static_cast<int>(rows), off.get(), off.get() + 1, 0, 64, st));
        note_launch();
        take_prefix_kernel<<<grid_for(rows * k, 256), 256, 0, st>>>(sorted.get(), rows, n, k, out + r0 * k);
        RBC_LAUNCHED();
    }
    return RBC_OK;
}

}  // namespace rbc
