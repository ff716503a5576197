// simt_scan.cu -- the fp32 SIMT filter with an exact fp64 re-rank: the L1 engine (north
// star: "L1 is an all-SIMT path"), and the L2 engine wherever the tensor-core scans do not
// pay (small problems, d > 128).
//
// Every (query, point) pair is evaluated once in fp32 on the FP32 pipe; only pairs whose
// fp32 distance can still reach the query's k best are recomputed with the reference
// arithmetic (common.cuh exact_dist: fp64, coordinate order, one rounding to fp32,
// metric.py:36-54) and enter an exact key64 top-k (brute_force.py:62-82).  The filter is
// rigorous, so the keys are the reference's bit for bit:
//
//   S  = fp32 sum of |a_k - b_k| (L1) or (a_k - b_k)^2 (L2, FMA), any summation order
//   |S - D| <= gamma_{d+1} D + d 2^-148       (D = the real-valued sum)
//   the reference's distance is D (1 +- u) (L1) or sqrt(D) (1 +- u) (L2) before ties,
//
// so a point with S > T = S_k (1 + (4 d + 16) 2^-24) + d 1e-35, S_k the k-th smallest
// fp32 sum seen so far, has a reference distance strictly above k already-seen points'
// and cannot be in the answer.  Points that pass are queued per thread (shared memory)
// and re-checked against the (tighter) bound once per tile before the exact fp64
// evaluation, so a warp pays for ~one exact distance per tile instead of one per lane.
//
// Work decomposition.  A CTA (256 threads) owns one work item: up to 256 queries and a
// contiguous range of point rows.  Point tiles are staged in shared memory with
// cp.async (two stages); every thread holds its query in registers and reads the tile
// rows as warp broadcasts.  When an item has fewer than 256 queries the point range is
// split over R = 256 / queries thread slices and the slices' exact top-k lists are
// merged at the end.
//   * dense items (bf_search, nearest representative, build assignment): all queries x
//     all rows, query blocks x point splits (splits merged by merge_parts);
//   * grouped items (one-shot search, search.py:114-120): queries sorted by nearest
//     representative, one item per (representative, 256 of its queries) x its s-list.
#include <cub/cub.cuh>

#include <atomic>

#include "common.cuh"
#include "index.cuh"
#include "kernels.cuh"
#include "tc_scan.cuh"

namespace rbc {

namespace {

constexpr int kST = 256;   // threads per CTA = most queries per work item
constexpr int kQLen = 8;   // pending candidates per thread (shared memory queue)

struct __align__(16) ScanItem {
    int32_t qbeg;  // first position in qorder
    int32_t qcnt;  // queries (<= kST x QPT)
    int32_t pbeg;  // first point row
    int32_t pcnt;  // point rows
};

struct SimtParams {
    const float *q;
    int64_t nq;
    int d;
    int d4;                  // row stride of the shared-memory tiles (d rounded up to 4)
    int tp;                  // points per tile
    const int32_t *qorder;   // grouped: query of each position
    const float *p;          // point rows [*][d]
    const int32_t *pid;      // id of each point row (nullptr: the row index)
    const ScanItem *items;   // grouped items (nullptr: dense)
    const int32_t *nitems;
    int64_t np;              // dense: point rows
    int64_t pchunk;          // dense: rows per split (< 2^31)
    int nqb;                 // dense: query blocks
    int qblk;                // dense: queries per block
    int k;
    uint64_t *out;           // [slot][nq][k]
};

__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// packed fp32 pairs (FADD2 / FFMA2 on sm_100)
__device__ __forceinline__ uint64_t f2u(float2 v) { return *reinterpret_cast<const uint64_t *>(&v); }
__device__ __forceinline__ float2 u2f(uint64_t v) { return *reinterpret_cast<const float2 *>(&v); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
    uint64_t r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(r);
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
    return u2f(r);
}

// two coordinates of one (query, point) pair into the pair accumulator acc
template <int METRIC>
__device__ __forceinline__ void acc2(float2 q, float2 x, float2 &acc) {
    const float2 t = sub2(q, x);
    if (METRIC == RBC_L2) {
        acc = fma2(t, t, acc);
    } else {
        acc.x += fabsf(t.x);
        acc.y += fabsf(t.y);
    }
}

// one fp32 sum into a running top-KT of fp32 sums; returns the new threshold T
template <int KT>
__device__ __forceinline__ float topk_push(float (&sv)[KT], float S, int k, float fac, float absl) {
    float x = S;
#pragma unroll
    for (int u = 0; u < KT; ++u) {
        const float lo = fminf(sv[u], x), hi = fmaxf(sv[u], x);
        sv[u] = lo;
        x = hi;
    }
    float kth = sv[KT - 1];
    if (KT != 1 && k != KT) {
#pragma unroll
        for (int u = 0; u < KT; ++u)
            if (u == k - 1) kth = sv[u];
    }
    return fmaf(kth, fac, absl);
}

// QPT queries per thread (each tile row read from shared memory once for all of them),
// DMAX >= d coordinates held in registers per query
template <int METRIC, int DMAX, int KT, int QPT>
__global__ void __launch_bounds__(kST) simt_scan_kernel(const SimtParams P) {
    extern __shared__ __align__(16) float smem[];
    // item
    int64_t qbeg, pbeg;
    int qcnt, pcnt;
    int slot = 0;
    if (P.items) {
        if (static_cast<int>(blockIdx.x) >= *P.nitems) return;
        const ScanItem it = P.items[blockIdx.x];
        qbeg = it.qbeg;
        qcnt = it.qcnt;
        pbeg = it.pbeg;
        pcnt = it.pcnt;
    } else {
        const int qb = static_cast<int>(blockIdx.x % P.nqb);
        slot = static_cast<int>(blockIdx.x / P.nqb);
        qbeg = static_cast<int64_t>(qb) * P.qblk;
        qcnt = static_cast<int>(min(static_cast<int64_t>(P.qblk), P.nq - qbeg));
        pbeg = static_cast<int64_t>(slot) * P.pchunk;
        pcnt = static_cast<int>(min(P.pchunk, P.np - pbeg));
    }
    const int d = P.d, d4 = P.d4, tp = P.tp, k = P.k;
    const int tid = threadIdx.x;
    // nqt query threads (QPT queries each) x R point slices; the slices' exact lists are
    // merged through shared memory at the end
    const int nqt = (qcnt + QPT - 1) / QPT;
    const int R = max(1, min(kST / nqt, kST / k));
    const bool active = tid < nqt * R;
    const int qslot = active ? tid % nqt : 0, slice = active ? tid / nqt : 0;
    int qpos[QPT];
    const float *qg[QPT];
    float2 qv[QPT][DMAX / 2];
#pragma unroll
    for (int u = 0; u < QPT; ++u) {
        qpos[u] = qslot + u * nqt;
        const int pos = qpos[u] < qcnt ? qpos[u] : qslot;  // a missing query repeats the thread's first
        const int64_t qi = P.qorder ? P.qorder[qbeg + pos] : qbeg + pos;
        qg[u] = P.q + qi * d;
#pragma unroll
        for (int c = 0; c < DMAX / 2; ++c)
            qv[u][c] = make_float2(2 * c < d ? __ldg(qg[u] + 2 * c) : 0.f, 2 * c + 1 < d ? __ldg(qg[u] + 2 * c + 1) : 0.f);
    }

    float *tiles = smem;                                              // [2][tp][d4]
    float *qs_s = smem + 2 * tp * d4;                                 // [kQLen][kST] pending fp32 sums
    uint32_t *qs_r = reinterpret_cast<uint32_t *>(qs_s + kQLen * kST);  // [kQLen][kST] (query << 31) | row
    // zero the pad columns once (cp.async writes only columns < d)
    if (d4 != d)
        for (int e = tid; e < 2 * tp; e += kST)
            for (int c = d; c < d4; ++c) tiles[e * d4 + c] = 0.f;

    const float fac = 1.0f + static_cast<float>(4 * d + 16) * (1.0f / 16777216.0f);
    const float absl = static_cast<float>(d) * 1e-35f;
    float sv[QPT][KT];
    uint64_t ek[QPT][KT];
    float T[QPT];
#pragma unroll
    for (int u = 0; u < QPT; ++u) {
        T[u] = __int_as_float(0x7f800000);
#pragma unroll
        for (int j = 0; j < KT; ++j) {
            sv[u][j] = __int_as_float(0x7f800000);
            ek[u][j] = kEmptyKey;
        }
    }
    int qn = 0;

    auto issue = [&](int t0, int buf) {
        const int tn = min(tp, pcnt - t0);
        const float *src = P.p + (pbeg + t0) * d;
        float *dst = tiles + buf * tp * d4;
        const int total = tn * d;
        for (int e = tid; e < total; e += kST) {
            const int r = e / d, c = e - r * d;
            cp_async4(dst + r * d4 + c, src + e);
        }
        cp_async_commit();
    };

    const int ntiles = (pcnt + tp - 1) / tp;
    __syncthreads();  // pad zeros before the first cp.async lands next to them
    if (ntiles > 0) issue(0, 0);
    for (int t = 0; t < ntiles; ++t) {
        const int buf = t & 1;
        if (t + 1 < ntiles) {
            issue((t + 1) * tp, buf ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        if (active) {
            const int t0 = t * tp;
            const int tn = min(tp, pcnt - t0);
            const float *tile = tiles + buf * tp * d4;
            // the inner loop leaves early only when the queue may overflow; the queue is drained
            // at one site (the exact fp64 evaluation is inlined once)
            int j = slice;
            for (;;) {
                for (; j < tn; j += R) {
                    const float4 *xr = reinterpret_cast<const float4 *>(tile + j * d4);
                    float2 acc[QPT][2];
#pragma unroll
                    for (int u = 0; u < QPT; ++u) acc[u][0] = acc[u][1] = make_float2(0.f, 0.f);
#pragma unroll
                    for (int c = 0; c < DMAX / 4; ++c) {
                        if (4 * c < d) {
                            const float4 x = xr[c];
#pragma unroll
                            for (int u = 0; u < QPT; ++u) {
                                acc2<METRIC>(qv[u][2 * c], make_float2(x.x, x.y), acc[u][0]);
                                acc2<METRIC>(qv[u][2 * c + 1], make_float2(x.z, x.w), acc[u][1]);
                            }
                        }
                    }
#pragma unroll
                    for (int u = 0; u < QPT; ++u) {
                        const float S = (acc[u][0].x + acc[u][1].x) + (acc[u][0].y + acc[u][1].y);
                        if (S < sv[u][KT - 1]) T[u] = topk_push<KT>(sv[u], S, k, fac, absl);
                        if (S <= T[u]) {
                            qs_s[qn * kST + tid] = S;
                            qs_r[qn * kST + tid] = (static_cast<uint32_t>(u) << 31) | static_cast<uint32_t>(t0 + j);
                            ++qn;
                        }
                    }
                    if (qn > kQLen - QPT) {
                        j += R;
                        break;
                    }
                }
                // exact fp64 evaluation of the queued points that can still qualify
                for (int e = 0; e < qn; ++e) {
                    const float s = qs_s[e * kST + tid];
                    const uint32_t rw = qs_r[e * kST + tid];
                    const int u = static_cast<int>(rw >> 31);
                    float Tu = T[0];
#pragma unroll
                    for (int v = 1; v < QPT; ++v)
                        if (u == v) Tu = T[v];
                    if (s <= Tu) {
                        const int64_t row = static_cast<int64_t>(rw & 0x7FFFFFFFu) + pbeg;
                        const uint32_t id = P.pid ? static_cast<uint32_t>(P.pid[row]) : static_cast<uint32_t>(row);
                        const float *qq = qg[0];
#pragma unroll
                        for (int v = 1; v < QPT; ++v)
                            if (u == v) qq = qg[v];
                        const uint64_t key = pack_key(exact_dist<METRIC>(qq, P.p + row * d, d), id);
#pragma unroll
                        for (int v = 0; v < QPT; ++v)
                            if (u == v && key < ek[v][KT - 1]) sorted_insert<KT>(ek[v], key);
                    }
                }
                qn = 0;
                if (j >= tn) break;
            }
        }
        __syncthreads();  // the buffer is refilled by the next issue
    }
    // merge the slices' exact lists (R > 1) and write the k best keys
    if (R == 1) {
        if (active)
#pragma unroll
            for (int u = 0; u < QPT; ++u)
                if (qpos[u] < qcnt) {
                    const int64_t qi = P.qorder ? P.qorder[qbeg + qpos[u]] : qbeg + qpos[u];
                    uint64_t *outq = P.out + (static_cast<int64_t>(slot) * P.nq + qi) * k;
#pragma unroll
                    for (int j = 0; j < KT; ++j)
                        if (j < k) outq[j] = ek[u][j];
                }
        return;
    }
    uint64_t *mk = reinterpret_cast<uint64_t *>(smem);  // [R][qcnt][k] (the tiles are done)
    if (active)
#pragma unroll
        for (int u = 0; u < QPT; ++u)
            if (qpos[u] < qcnt)
#pragma unroll
                for (int j = 0; j < KT; ++j)
                    if (j < k) mk[(static_cast<int64_t>(slice) * qcnt + qpos[u]) * k + j] = ek[u][j];
    __syncthreads();
    for (int qp = tid; qp < qcnt; qp += kST) {
        uint64_t best[KT];
#pragma unroll
        for (int j = 0; j < KT; ++j) best[j] = kEmptyKey;
        for (int s = 0; s < R; ++s)
            for (int j = 0; j < k; ++j) {
                const uint64_t key = mk[(static_cast<int64_t>(s) * qcnt + qp) * k + j];
                if (key >= best[KT - 1]) break;  // each slice's list ascends
                sorted_insert<KT>(best, key);
            }
        const int64_t qi = P.qorder ? P.qorder[qbeg + qp] : qbeg + qp;
        uint64_t *outq = P.out + (static_cast<int64_t>(slot) * P.nq + qi) * k;
#pragma unroll
        for (int j = 0; j < KT; ++j)
            if (j < k) outq[j] = best[j];
    }
}

// ---- one-shot grouping: queries by nearest representative --------------------------------
__global__ void near_hist_kernel(const uint64_t *__restrict__ near, int64_t nq, int32_t *__restrict__ cnt) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < nq) atomicAdd(&cnt[key_id(near[i])], 1);
}

__global__ void near_chunks_kernel(const int32_t *__restrict__ cnt, int64_t nr, int qb, int32_t *__restrict__ nchunk) {
    const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (r < nr) nchunk[r] = (cnt[r] + qb - 1) / qb;
}

__global__ void near_scatter_kernel(const uint64_t *__restrict__ near, int64_t nq, const int32_t *__restrict__ start,
                                    int32_t *__restrict__ fill, int32_t *__restrict__ qorder) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= nq) return;
    const uint32_t r = key_id(near[i]);
    qorder[start[r] + atomicAdd(&fill[r], 1)] = static_cast<int32_t>(i);
}

__global__ void near_items_kernel(const int32_t *__restrict__ cnt, const int32_t *__restrict__ start,
                                  const int32_t *__restrict__ istart, int64_t nr, int s, int qb,
                                  ScanItem *__restrict__ items, int32_t *__restrict__ nitems) {
    const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (r >= nr) return;
    const int c = cnt[r];
    const int nc = (c + qb - 1) / qb;
    for (int j = 0; j < nc; ++j) {
        ScanItem it;
        it.qbeg = start[r] + j * qb;
        it.qcnt = min(qb, c - j * qb);
        it.pbeg = static_cast<int32_t>(r * s);
        it.pcnt = s;
        items[istart[r] + j] = it;
    }
    if (r == nr - 1) *nitems = istart[r] + nc;
}

int simt_dmax(int d) { return d <= 24 ? 24 : d <= 32 ? 32 : d <= 64 ? 64 : 128; }
int simt_kt(int k) { return k <= 1 ? 1 : k <= 4 ? 4 : k <= 16 ? 16 : 32; }
// two queries per thread where their coordinates fit the registers (and the merge buffer
// of two queries x k keys per thread fits shared memory)
int simt_qpt(int d, int k) { return d <= 32 && k <= 16 ? 2 : 1; }

int simt_tp(int d4) { return d4 <= 64 ? 128 : 64; }

size_t simt_smem(int d4, int tp, int k, int qpt) {
    const size_t tiles = 2 * static_cast<size_t>(tp) * d4 * sizeof(float);
    const size_t merge = static_cast<size_t>(kST) * qpt * k * sizeof(uint64_t);
    return (tiles > merge ? tiles : merge) + kQLen * kST * (sizeof(float) + sizeof(int32_t));
}

template <int METRIC, int DMAX, int KT, int QPT>
int launch_kt(const SimtParams &P, unsigned grid, size_t smem, cudaStream_t st) {
    auto *fn = simt_scan_kernel<METRIC, DMAX, KT, QPT>;
    if (smem > 48 * 1024)
        RBC_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    fn<<<grid, kST, smem, st>>>(P);
    RBC_LAUNCHED();
    return RBC_OK;
}

template <int METRIC, int DMAX>
int launch_dmax(const SimtParams &P, unsigned grid, size_t smem, cudaStream_t st) {
    if constexpr (DMAX <= 32) {
        if (simt_qpt(P.d, P.k) == 2) {
            switch (simt_kt(P.k)) {
                case 1: return launch_kt<METRIC, DMAX, 1, 2>(P, grid, smem, st);
                case 4: return launch_kt<METRIC, DMAX, 4, 2>(P, grid, smem, st);
                default: return launch_kt<METRIC, DMAX, 16, 2>(P, grid, smem, st);
            }
        }
        return launch_kt<METRIC, DMAX, 32, 1>(P, grid, smem, st);
    } else {
        switch (simt_kt(P.k)) {
            case 1: return launch_kt<METRIC, DMAX, 1, 1>(P, grid, smem, st);
            case 4: return launch_kt<METRIC, DMAX, 4, 1>(P, grid, smem, st);
            case 16: return launch_kt<METRIC, DMAX, 16, 1>(P, grid, smem, st);
            default: return launch_kt<METRIC, DMAX, 32, 1>(P, grid, smem, st);
        }
    }
}

template <int METRIC>
int launch_metric(const SimtParams &P, unsigned grid, size_t smem, cudaStream_t st) {
    switch (simt_dmax(P.d)) {
        case 24: return launch_dmax<METRIC, 24>(P, grid, smem, st);
        case 32: return launch_dmax<METRIC, 32>(P, grid, smem, st);
        case 64: return launch_dmax<METRIC, 64>(P, grid, smem, st);
        default: return launch_dmax<METRIC, 128>(P, grid, smem, st);
    }
}

std::atomic<int64_t> g_simt_calls{0};

int simt_launch(SimtParams P, int metric, unsigned grid, cudaStream_t st) {
    g_simt_calls.fetch_add(1);
    P.d4 = (P.d + 3) & ~3;
    P.tp = simt_tp(P.d4);
    const size_t smem = simt_smem(P.d4, P.tp, P.k, simt_qpt(P.d, P.k));
    return metric == RBC_L2 ? launch_metric<RBC_L2>(P, grid, smem, st) : launch_metric<RBC_L1>(P, grid, smem, st);
}

}  // namespace

bool simt_supported(int d, int k) { return d >= 1 && d <= 128 && k >= 1 && k <= 32; }

bool simt_one_shot_supported(const rbc_index *idx, int64_t nq, int k) {
    return idx->kind == 1 && idx->xp != nullptr && simt_supported(idx->d, k) && k <= idx->s &&
           idx->nr * static_cast<int64_t>(idx->s) < (int64_t(1) << 31) && nq < (int64_t(1) << 31) &&
           nq * idx->s >= simt_min_pairs();
}

// k nearest keys (ascending) of every q row over the rows of x; ids = row index (pid
// nullptr) or pid[row]
int simt_dense_topk(const float *q, int64_t nq, const float *x, int64_t n, int d, int metric, int k,
                    const int32_t *pid, uint64_t *keys, cudaStream_t st) {
    if (nq == 0) return RBC_OK;
    if (!simt_supported(d, k)) return fail(RBC_EINVAL, "simt scan: unsupported d or k");
    // queries per CTA: kST x QPT / Rt (Rt point slices per query thread), the fewest slices
    // giving >= ~600 CTAs; point splits (merged by merge_parts) only when the queries alone
    // cannot fill the GPU
    const int qpt = simt_qpt(d, k);
    int qblk = kST * qpt;
    while (qblk > 32 * qpt && (nq + qblk - 1) / qblk < 600 && qblk / 2 >= 32 * qpt && kST * qpt / (qblk / 2) <= kST / k)
        qblk /= 2;
    const int64_t nqb = (nq + qblk - 1) / qblk;
    int64_t splits = (600 + nqb - 1) / nqb;
    const int64_t max_splits = (n + 2047) / 2048;
    if (splits > max_splits) splits = max_splits;
    if (splits < 1) splits = 1;
    const int64_t pchunk = (n + splits - 1) / splits;
    splits = (n + pchunk - 1) / pchunk;
    if (nqb * splits > 0x7FFFFFFF || n >= (int64_t(1) << 31))
        return fail(RBC_EINVAL, "simt scan: problem too large for one call");
    DevBuf<uint64_t> part;
    if (splits > 1) RBC_CHECK(part.alloc(splits * nq * k, st));
    SimtParams P{};
    P.q = q;
    P.nq = nq;
    P.d = d;
    P.p = x;
    P.pid = pid;
    P.np = n;
    P.pchunk = pchunk;
    P.nqb = static_cast<int>(nqb);
    P.qblk = qblk;
    P.k = k;
    P.out = splits > 1 ? part.get() : keys;
    RBC_CHECK(simt_launch(P, metric, static_cast<unsigned>(nqb * splits), st));
    if (splits > 1) RBC_CHECK(merge_parts(part.get(), static_cast<int>(splits), nq, k, k, keys, st));
    return RBC_OK;
}

// one-shot list scan: query i scans the s-list of its nearest representative key_id(near[i])
// (rows [p s, p s + s) of idx->xp, ids idx->lists)
int simt_one_shot_scan(const rbc_index *idx, const float *q, int64_t nq, int k, const uint64_t *near, uint64_t *keys,
                       cudaStream_t st) {
    if (nq == 0) return RBC_OK;
    if (!simt_one_shot_supported(idx, nq, k)) return fail(RBC_EINVAL, "simt one-shot scan: unsupported");
    const int64_t nr = idx->nr;
    DevBuf<int32_t> cnt, fill, start, nchunk, istart, qorder, nitems;
    DevBuf<ScanItem> items;
    RBC_CHECK(cnt.alloc(nr, st));
    RBC_CHECK(fill.alloc(nr, st));
    RBC_CHECK(start.alloc(nr, st));
    RBC_CHECK(nchunk.alloc(nr, st));
    RBC_CHECK(istart.alloc(nr, st));
    RBC_CHECK(qorder.alloc(nq, st));
    RBC_CHECK(nitems.alloc(1, st));
    const int qb = kST * simt_qpt(idx->d, k);
    const int64_t max_items = std::min<int64_t>(nr, nq) + nq / qb + 1;
    RBC_CHECK(items.alloc(max_items, st));
    RBC_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(int32_t) * nr, st));
    RBC_CUDA(cudaMemsetAsync(fill.get(), 0, sizeof(int32_t) * nr, st));
    near_hist_kernel<<<grid_for(nq, 256), 256, 0, st>>>(near, nq, cnt.get());
    RBC_LAUNCHED();
    near_chunks_kernel<<<grid_for(nr, 256), 256, 0, st>>>(cnt.get(), nr, qb, nchunk.get());
    RBC_LAUNCHED();
    size_t tb = 0, tb2 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.get(), start.get(), nr, st);
    cub::DeviceScan::ExclusiveSum(nullptr, tb2, nchunk.get(), istart.get(), nr, st);
    DevBuf<unsigned char> tmp;
    RBC_CHECK(tmp.alloc(std::max(tb, tb2), st));
    RBC_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb, cnt.get(), start.get(), nr, st));
    RBC_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb2, nchunk.get(), istart.get(), nr, st));
    note_launch(2);
    near_scatter_kernel<<<grid_for(nq, 256), 256, 0, st>>>(near, nq, start.get(), fill.get(), qorder.get());
    RBC_LAUNCHED();
    near_items_kernel<<<grid_for(nr, 256), 256, 0, st>>>(cnt.get(), start.get(), istart.get(), nr, idx->s, qb,
                                                        items.get(), nitems.get());
    RBC_LAUNCHED();
    SimtParams P{};
    P.q = q;
    P.nq = nq;
    P.d = idx->d;
    P.qorder = qorder.get();
    P.p = idx->xp;
    P.pid = idx->lists;
    P.items = items.get();
    P.nitems = nitems.get();
    P.k = k;
    P.out = keys;
    return simt_launch(P, idx->metric, static_cast<unsigned>(max_items), st);
}

}  // namespace rbc

extern "C" int64_t rbc_simt_scan_calls(void) { return rbc::g_simt_calls.load(); }
