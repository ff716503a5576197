// simt_scan.cu -- the fp32 SIMT filter with an exact fp64 re-rank: the L1 engine (north
// star: "L1 is an all-SIMT path"), and the L2 engine wherever the tensor-core scans do not
// apply (d > 128) or do not pay (small scans).
//
// Every (query, point) pair is evaluated once in fp32; only pairs whose fp32 distance can
// still reach the query's k best are recomputed with the reference arithmetic
// (common.cuh exact_dist: fp64, coordinate order, one rounding to fp32, metric.py:36-54)
// and enter an exact key64 top-k (brute_force.py:62-82).  The filter is rigorous, so the
// keys are the reference's bit for bit:
//
//   S  = fp32 sum of |a_k - b_k| (L1) or (a_k - b_k)^2 (L2, FMA), any summation order
//   |S - D| <= gamma_{d+1} D + d 2^-148       (D = the real-valued sum)
//   the reference's distance is D (1 +- u) (L1) or sqrt(D) (1 +- u) (L2) before ties,
//
// so a point with S > T = S_k (1 + (4 d + 16) 2^-24) + d 1e-35, S_k the k-th smallest
// fp32 sum seen so far, has a reference distance strictly above k already-seen points'
// and cannot be in the answer.
//
// Work decomposition.  A CTA (8 warps) owns one work item: up to 32 x QPT queries (lane
// l holds queries l, l + 32, ..., coordinates in registers) and a range of point rows,
// staged through shared memory in tiles (cp.async, two stages) with a 16-byte aligned row
// stride d4 = d rounded up to 4 (zero padded; |0 - 0| adds nothing).  Warp w scans tile
// rows w, w + 8, ...: every lane of a warp reads the same row (a shared-memory broadcast)
// and uses it for QPT queries.  After each tile the warps publish their per-query bounds
// and all adopt the minimum (any warp's k-th smallest sum bounds the union's), so the
// eight-way split filters as tightly as one scan; the warps' exact lists are merged at
// the end.
//   * dense items (bf_search, nearest representative, build assignment): query chunks x
//     point splits (splits merged by merge_parts);
//   * grouped items (one-shot search, search.py:114-120): queries sorted by nearest
//     representative, one item per (representative, chunk of its queries) x its s-list.
// Points that pass the filter are queued per lane in shared memory and drained after the
// bound exchange, so most stale candidates are dropped before the exact fp64 evaluation.
#include <cub/cub.cuh>

#include <atomic>

#include "common.cuh"
#include "index.cuh"
#include "kernels.cuh"
#include "tc_scan.cuh"

namespace rbc {

namespace {

constexpr int kW = 8;        // warps per CTA (point slices)
constexpr int kT = 32 * kW;
constexpr int kQLen = 8;     // queued candidates per lane

struct __align__(16) ScanItem {
    int32_t qbeg;  // first position in qorder
    int32_t qcnt;  // queries (<= 32 x QPT)
    int32_t pbeg;  // first point row
    int32_t pcnt;  // point rows
};

struct SimtParams {
    const float *q;          // queries [nq][d]
    int64_t nq;
    int d;
    int d4;                  // row stride of p (d rounded up to 4)
    int tp;                  // rows per tile
    const int32_t *qorder;   // grouped: query of each sorted position
    const ScanItem *items;   // grouped items (nullptr: dense)
    const int32_t *nitems;
    const float *p;          // point rows [*][d4], 16-byte aligned
    const int32_t *pid;      // id of each point row (nullptr: the row index)
    int64_t nqc;             // dense: query chunks
    int64_t np;              // dense: point rows
    int64_t pchunk;          // dense: rows per split (< 2^31)
    int k;
    int qpt;                 // queries per lane (host side: selects the instantiation)
    uint64_t *out;           // [split][nq][k]
};
// segment items (simt_seg_kernel only; a separate parameter block keeps simt_tile_kernel's as it was)
struct SimtSegParams : SimtParams {
    const int32_t *qcut;     // rows of the item each position scans (nullptr: not segment items)
    const int64_t *qout;     // output row of each position
    const float *qthr;       // initial fp32 bound of each position
};

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

// one fp32 sum into the running top-KT of fp32 sums; returns the new threshold T
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

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int METRIC, int DMAX, int KT, int QPT>
__global__ void __launch_bounds__(kT, DMAX * QPT <= 64 ? 2 : 1) simt_tile_kernel(const SimtParams P) {
    extern __shared__ __align__(16) float smem[];
    int64_t qbeg, pbeg;
    int qcnt, pcnt;
    int64_t slot = 0;
    if (P.items) {
        if (static_cast<int>(blockIdx.x) >= *P.nitems) return;
        const ScanItem it = P.items[blockIdx.x];
        qbeg = it.qbeg;
        qcnt = it.qcnt;
        pbeg = it.pbeg;
        pcnt = it.pcnt;
    } else {
        const int64_t chunk = blockIdx.x % P.nqc;
        slot = blockIdx.x / P.nqc;
        qbeg = chunk * 32 * QPT;
        qcnt = static_cast<int>(min(static_cast<int64_t>(32 * QPT), P.nq - qbeg));
        pbeg = slot * P.pchunk;
        pcnt = static_cast<int>(min(P.pchunk, P.np - pbeg));
    }
    const int d = P.d, d4 = P.d4, tp = P.tp, k = P.k;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    float *tiles = smem;                                            // [2][tp][d4]
    float *tsh = smem + 2 * tp * d4;                                // [kW][32 QPT] published bounds
    float *qs_s = tsh + kW * 32 * QPT;                              // [kQLen][kT] queued sums
    uint32_t *qs_r = reinterpret_cast<uint32_t *>(qs_s + kQLen * kT);  // [kQLen][kT] (u << 28) | row
    const float *qg[QPT];
    float2 qv[QPT][DMAX / 2];
#pragma unroll
    for (int u = 0; u < QPT; ++u) {
        const int pos = 32 * u + lane < qcnt ? 32 * u + lane : 0;  // a missing query repeats the first
        const int64_t qi = P.qorder ? P.qorder[qbeg + pos] : qbeg + pos;
        qg[u] = P.q + qi * d;
#pragma unroll
        for (int c = 0; c < DMAX / 2; ++c)
            qv[u][c] = make_float2(2 * c < d ? __ldg(qg[u] + 2 * c) : 0.f, 2 * c + 1 < d ? __ldg(qg[u] + 2 * c + 1) : 0.f);
    }
    const float fac = 1.0f + static_cast<float>(4 * d + 16) * (1.0f / 16777216.0f);
    const float absl = static_cast<float>(d) * 1e-35f;
    float sv[QPT][KT], T[QPT];
    uint64_t ek[QPT][KT];
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
    // exact fp64 evaluation of the queued points that still qualify
    auto drain = [&]() {
        for (int e = 0; e < qn; ++e) {
            const float sq = qs_s[e * kT + tid];
            const uint32_t rw = qs_r[e * kT + tid];
            const int u = static_cast<int>(rw >> 28);
            float Tu = T[0];
            const float *qq = qg[0];
#pragma unroll
            for (int v = 1; v < QPT; ++v)
                if (u == v) {
                    Tu = T[v];
                    qq = qg[v];
                }
            if (sq <= Tu) {
                const int64_t row = pbeg + static_cast<int64_t>(rw & 0x0FFFFFFFu);
                const uint32_t id = P.pid ? static_cast<uint32_t>(P.pid[row]) : static_cast<uint32_t>(row);
                const uint64_t key = pack_key(exact_dist<METRIC>(qq, P.p + row * d4, d), id);
#pragma unroll
                for (int v = 0; v < QPT; ++v)
                    if (u == v && key < ek[v][KT - 1]) sorted_insert<KT>(ek[v], key);
            }
        }
        qn = 0;
    };
    // tile copies: the tile's rows are contiguous and 16-byte aligned (padded stride d4)
    auto tile_rows = [&](int t0) { return min(t0 == 0 ? 2 * kW : tp, pcnt - t0); };
    auto issue = [&](int t0, int buf) {
        const int tn = tile_rows(t0);
        const float4 *src = reinterpret_cast<const float4 *>(P.p + (pbeg + t0) * d4);
        float4 *dst = reinterpret_cast<float4 *>(tiles + buf * tp * d4);
        for (int e = tid; e < tn * (d4 >> 2); e += kT) cp_async16(dst + e, src + e);
        cp_async_commit();
    };

    // tiles: a short first one (two rows per warp: after its bound exchange every query
    // starts from the best of 16 rows, so the later tiles rarely queue a candidate), then
    // tp rows each
    int t = 0;
    if (pcnt > 0) issue(0, 0);
    for (int t0 = 0; t0 < pcnt; t0 += tile_rows(t0), ++t) {
        const int buf = t & 1, tn = tile_rows(t0);
        if (t0 + tn < pcnt) {
            issue(t0 + tn, buf ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const float *tile = tiles + buf * tp * d4;
        // kRows tile rows per step (a warp's rows j, j + kW, ...): every row's loads are issued
        // before any arithmetic (independent registers, predicated instead of branched), so the
        // shared-memory latency overlaps across rows and chunks
        constexpr int kRowsStep = DMAX * (QPT + 2) <= 128 ? 2 : 1;
        for (int j = warp; j < tn; j += kRowsStep * kW) {
            float4 xs[kRowsStep][DMAX / 4];
#pragma unroll
            for (int rr = 0; rr < kRowsStep; ++rr) {
                const int jr = j + rr * kW < tn ? j + rr * kW : j;
                const float4 *xr = reinterpret_cast<const float4 *>(tile + jr * d4);
#pragma unroll
                for (int c = 0; c < DMAX / 4; ++c) xs[rr][c] = 4 * c < d ? xr[c] : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int rr = 0; rr < kRowsStep; ++rr) {
                if (j + rr * kW >= tn) break;  // warp-uniform
                float2 acc[QPT][2];
#pragma unroll
                for (int u = 0; u < QPT; ++u) acc[u][0] = acc[u][1] = make_float2(0.f, 0.f);
#pragma unroll
                for (int c = 0; c < DMAX / 4; ++c) {
#pragma unroll
                    for (int u = 0; u < QPT; ++u) {
                        acc2<METRIC>(qv[u][2 * c], make_float2(xs[rr][c].x, xs[rr][c].y), acc[u][0]);
                        acc2<METRIC>(qv[u][2 * c + 1], make_float2(xs[rr][c].z, xs[rr][c].w), acc[u][1]);
                    }
                }
#pragma unroll
                for (int u = 0; u < QPT; ++u) {
                    const float S = (acc[u][0].x + acc[u][1].x) + (acc[u][0].y + acc[u][1].y);
                    if (S < sv[u][KT - 1]) T[u] = fminf(T[u], topk_push<KT>(sv[u], S, k, fac, absl));
                    if (S <= T[u]) {
                        qs_s[qn * kT + tid] = S;
                        qs_r[qn * kT + tid] = (static_cast<uint32_t>(u) << 28) | static_cast<uint32_t>(t0 + j + rr * kW);
                        ++qn;
                    }
                }
                if (__any_sync(0xffffffffu, qn > kQLen - QPT)) drain();
            }
        }
        // bound exchange: every warp adopts the smallest published bound of each query
#pragma unroll
        for (int u = 0; u < QPT; ++u) tsh[warp * 32 * QPT + 32 * u + lane] = T[u];
        __syncthreads();  // (also: the buffer is refilled by the next issue)
#pragma unroll
        for (int u = 0; u < QPT; ++u) {
            float m = T[u];
#pragma unroll
            for (int w = 0; w < kW; ++w) m = fminf(m, tsh[w * 32 * QPT + 32 * u + lane]);
            T[u] = m;
        }
        drain();
    }
    // merge the warps' exact lists: mk[w][pos][k] (the tiles are done)
    __syncthreads();
    uint64_t *mk = reinterpret_cast<uint64_t *>(smem);
#pragma unroll
    for (int u = 0; u < QPT; ++u)
        if (32 * u + lane < qcnt)
#pragma unroll
            for (int j = 0; j < KT; ++j)
                if (j < k) mk[(static_cast<int64_t>(warp) * qcnt + 32 * u + lane) * k + j] = ek[u][j];
    __syncthreads();
    for (int qp = tid; qp < qcnt; qp += kT) {
        uint64_t best[KT];
#pragma unroll
        for (int j = 0; j < KT; ++j) best[j] = kEmptyKey;
        for (int w = 0; w < kW; ++w)
            for (int j = 0; j < k; ++j) {
                const uint64_t key = mk[(static_cast<int64_t>(w) * qcnt + qp) * k + j];
                if (key >= best[KT - 1]) break;  // each warp's list ascends
                sorted_insert<KT>(best, key);
            }
        const int64_t qi = P.qorder ? P.qorder[qbeg + qp] : qbeg + qp;
        uint64_t *outq = P.out + (slot * P.nq + qi) * k;
#pragma unroll
        for (int j = 0; j < KT; ++j)
            if (j < k) outq[j] = best[j];
    }
}

// The same scan over segment items (exact-search stage 2, simt_exact_stage2): per-position
// cutoffs, output rows and gamma-seeded bounds.  A separate kernel: folding these into
// simt_tile_kernel changed its code generation and cost the dense and one-shot scans ~10%.
template <int METRIC, int DMAX, int KT, int QPT>
__global__ void __launch_bounds__(kT, DMAX * QPT <= 64 ? 2 : 1) simt_seg_kernel(const SimtSegParams P) {
    constexpr bool SEG = true;
    extern __shared__ __align__(16) float smem[];
    int64_t qbeg, pbeg;
    int qcnt, pcnt;
    int64_t slot = 0;
    if (P.items) {
        if (static_cast<int>(blockIdx.x) >= *P.nitems) return;
        const ScanItem it = P.items[blockIdx.x];
        qbeg = it.qbeg;
        qcnt = it.qcnt;
        pbeg = it.pbeg;
        pcnt = it.pcnt;
    } else {
        const int64_t chunk = blockIdx.x % P.nqc;
        slot = blockIdx.x / P.nqc;
        qbeg = chunk * 32 * QPT;
        qcnt = static_cast<int>(min(static_cast<int64_t>(32 * QPT), P.nq - qbeg));
        pbeg = slot * P.pchunk;
        pcnt = static_cast<int>(min(P.pchunk, P.np - pbeg));
    }
    const int d = P.d, d4 = P.d4, tp = P.tp, k = P.k;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    float *tiles = smem;                                            // [2][tp][d4]
    float *tsh = smem + 2 * tp * d4;                                // [kW][32 QPT] published bounds
    float *qs_s = tsh + kW * 32 * QPT;                              // [kQLen][kT] queued sums
    uint32_t *qs_r = reinterpret_cast<uint32_t *>(qs_s + kQLen * kT);  // [kQLen][kT] (u << 28) | row
    const float *qg[QPT];
    float2 qv[QPT][DMAX / 2];
    int lim[SEG ? QPT : 1];  // segment items: rows each position scans (its list's cutoff)
#pragma unroll
    for (int u = 0; u < QPT; ++u) {
        const int pos = 32 * u + lane < qcnt ? 32 * u + lane : 0;  // a missing query repeats the first
        const int64_t qi = P.qorder ? P.qorder[qbeg + pos] : qbeg + pos;
        if constexpr (SEG) lim[u] = P.qcut[qbeg + pos];
        qg[u] = P.q + qi * d;
#pragma unroll
        for (int c = 0; c < DMAX / 2; ++c)
            qv[u][c] = make_float2(2 * c < d ? __ldg(qg[u] + 2 * c) : 0.f, 2 * c + 1 < d ? __ldg(qg[u] + 2 * c + 1) : 0.f);
    }
    const float fac = 1.0f + static_cast<float>(4 * d + 16) * (1.0f / 16777216.0f);
    const float absl = static_cast<float>(d) * 1e-35f;
    float sv[QPT][KT], T[QPT];
    uint64_t ek[QPT][KT];
#pragma unroll
    for (int u = 0; u < QPT; ++u) {
        T[u] = __int_as_float(0x7f800000);
        if constexpr (SEG) T[u] = P.qthr[qbeg + (32 * u + lane < qcnt ? 32 * u + lane : 0)];
#pragma unroll
        for (int j = 0; j < KT; ++j) {
            sv[u][j] = __int_as_float(0x7f800000);
            ek[u][j] = kEmptyKey;
        }
    }
    int qn = 0;
    // exact fp64 evaluation of the queued points that still qualify
    auto drain = [&]() {
        for (int e = 0; e < qn; ++e) {
            const float sq = qs_s[e * kT + tid];
            const uint32_t rw = qs_r[e * kT + tid];
            const int u = static_cast<int>(rw >> 28);
            float Tu = T[0];
            const float *qq = qg[0];
#pragma unroll
            for (int v = 1; v < QPT; ++v)
                if (u == v) {
                    Tu = T[v];
                    qq = qg[v];
                }
            if (sq <= Tu) {
                const int64_t row = pbeg + static_cast<int64_t>(rw & 0x0FFFFFFFu);
                const uint32_t id = P.pid ? static_cast<uint32_t>(P.pid[row]) : static_cast<uint32_t>(row);
                const uint64_t key = pack_key(exact_dist<METRIC>(qq, P.p + row * d4, d), id);
#pragma unroll
                for (int v = 0; v < QPT; ++v)
                    if (u == v && key < ek[v][KT - 1]) sorted_insert<KT>(ek[v], key);
            }
        }
        qn = 0;
    };
    // tile copies: the tile's rows are contiguous and 16-byte aligned (padded stride d4)
    auto tile_rows = [&](int t0) { return min(t0 == 0 ? 2 * kW : tp, pcnt - t0); };
    auto issue = [&](int t0, int buf) {
        const int tn = tile_rows(t0);
        const float4 *src = reinterpret_cast<const float4 *>(P.p + (pbeg + t0) * d4);
        float4 *dst = reinterpret_cast<float4 *>(tiles + buf * tp * d4);
        for (int e = tid; e < tn * (d4 >> 2); e += kT) cp_async16(dst + e, src + e);
        cp_async_commit();
    };

    // tiles: a short first one (two rows per warp: after its bound exchange every query
    // starts from the best of 16 rows, so the later tiles rarely queue a candidate), then
    // tp rows each
    int t = 0;
    if (pcnt > 0) issue(0, 0);
    for (int t0 = 0; t0 < pcnt; t0 += tile_rows(t0), ++t) {
        const int buf = t & 1, tn = tile_rows(t0);
        if (t0 + tn < pcnt) {
            issue(t0 + tn, buf ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const float *tile = tiles + buf * tp * d4;
        // kRows tile rows per step (a warp's rows j, j + kW, ...): every row's loads are issued
        // before any arithmetic (independent registers, predicated instead of branched), so the
        // shared-memory latency overlaps across rows and chunks
        constexpr int kRowsStep = DMAX * (QPT + 2) <= 128 ? 2 : 1;
        for (int j = warp; j < tn; j += kRowsStep * kW) {
            float4 xs[kRowsStep][DMAX / 4];
#pragma unroll
            for (int rr = 0; rr < kRowsStep; ++rr) {
                const int jr = j + rr * kW < tn ? j + rr * kW : j;
                const float4 *xr = reinterpret_cast<const float4 *>(tile + jr * d4);
#pragma unroll
                for (int c = 0; c < DMAX / 4; ++c) xs[rr][c] = 4 * c < d ? xr[c] : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int rr = 0; rr < kRowsStep; ++rr) {
                if (j + rr * kW >= tn) break;  // warp-uniform
                float2 acc[QPT][2];
#pragma unroll
                for (int u = 0; u < QPT; ++u) acc[u][0] = acc[u][1] = make_float2(0.f, 0.f);
#pragma unroll
                for (int c = 0; c < DMAX / 4; ++c) {
#pragma unroll
                    for (int u = 0; u < QPT; ++u) {
                        acc2<METRIC>(qv[u][2 * c], make_float2(xs[rr][c].x, xs[rr][c].y), acc[u][0]);
                        acc2<METRIC>(qv[u][2 * c + 1], make_float2(xs[rr][c].z, xs[rr][c].w), acc[u][1]);
                    }
                }
#pragma unroll
                for (int u = 0; u < QPT; ++u) {
                    const float S = (acc[u][0].x + acc[u][1].x) + (acc[u][0].y + acc[u][1].y);
                    if constexpr (SEG) {  // past its cutoff: the row is not a candidate of this position
                        if (t0 + j + rr * kW >= lim[u]) continue;
                    }
                    if (S < sv[u][KT - 1]) T[u] = fminf(T[u], topk_push<KT>(sv[u], S, k, fac, absl));
                    if (S <= T[u]) {
                        qs_s[qn * kT + tid] = S;
                        qs_r[qn * kT + tid] = (static_cast<uint32_t>(u) << 28) | static_cast<uint32_t>(t0 + j + rr * kW);
                        ++qn;
                    }
                }
                if (__any_sync(0xffffffffu, qn > kQLen - QPT)) drain();
            }
        }
        // bound exchange: every warp adopts the smallest published bound of each query
#pragma unroll
        for (int u = 0; u < QPT; ++u) tsh[warp * 32 * QPT + 32 * u + lane] = T[u];
        __syncthreads();  // (also: the buffer is refilled by the next issue)
#pragma unroll
        for (int u = 0; u < QPT; ++u) {
            float m = T[u];
#pragma unroll
            for (int w = 0; w < kW; ++w) m = fminf(m, tsh[w * 32 * QPT + 32 * u + lane]);
            T[u] = m;
        }
        drain();
    }
    // merge the warps' exact lists: mk[w][pos][k] (the tiles are done)
    __syncthreads();
    uint64_t *mk = reinterpret_cast<uint64_t *>(smem);
#pragma unroll
    for (int u = 0; u < QPT; ++u)
        if (32 * u + lane < qcnt)
#pragma unroll
            for (int j = 0; j < KT; ++j)
                if (j < k) mk[(static_cast<int64_t>(warp) * qcnt + 32 * u + lane) * k + j] = ek[u][j];
    __syncthreads();
    for (int qp = tid; qp < qcnt; qp += kT) {
        uint64_t best[KT];
#pragma unroll
        for (int j = 0; j < KT; ++j) best[j] = kEmptyKey;
        for (int w = 0; w < kW; ++w)
            for (int j = 0; j < k; ++j) {
                const uint64_t key = mk[(static_cast<int64_t>(w) * qcnt + qp) * k + j];
                if (key >= best[KT - 1]) break;  // each warp's list ascends
                sorted_insert<KT>(best, key);
            }
        int64_t qi;
        if constexpr (SEG) qi = P.qout[qbeg + qp];
        else qi = P.qorder ? P.qorder[qbeg + qp] : qbeg + qp;
        uint64_t *outq = P.out + (slot * P.nq + qi) * k;
#pragma unroll
        for (int j = 0; j < KT; ++j)
            if (j < k) outq[j] = best[j];
    }
}

// ---- one-shot grouping: queries sorted by nearest representative --------------------------
__global__ void near_hist_kernel(const uint64_t *__restrict__ near, int64_t nq, int32_t *__restrict__ cnt) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < nq) atomicAdd(&cnt[key_id(near[i])], 1);
}

__global__ void near_scatter_kernel(const uint64_t *__restrict__ near, int64_t nq, const int32_t *__restrict__ start,
                                    int32_t *__restrict__ fill, int32_t *__restrict__ qorder) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= nq) return;
    const uint32_t r = key_id(near[i]);
    qorder[start[r] + atomicAdd(&fill[r], 1)] = static_cast<int32_t>(i);
}

// rows [rows][d] -> [rows][d4] (zero padded), optionally gathered: src row = ids[r]
__global__ void pad_rows_kernel(const float *__restrict__ src, const int32_t *__restrict__ ids, int64_t rows, int d,
                                int d4, float *__restrict__ dst) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < rows * d4;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = t / d4;
        const int c = static_cast<int>(t - r * d4);
        const int64_t sr = ids ? ids[r] : r;
        dst[t] = c < d ? src[sr * d + c] : 0.f;
    }
}

__global__ void near_chunks_kernel(const int32_t *__restrict__ cnt, int64_t nr, int qb, int32_t *__restrict__ nchunk) {
    const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (r < nr) nchunk[r] = (cnt[r] + qb - 1) / qb;
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

// ---- exact-search stage 2 on the SIMT filter (search.py:183-186): surviving segments grouped by list --
__global__ void seg_query_kernel(const int64_t *__restrict__ seg_off, const int32_t *__restrict__ nseg, int64_t nq,
                                 const int32_t *__restrict__ seg_list, int32_t *__restrict__ seg_q,
                                 uint32_t *__restrict__ key, int32_t *__restrict__ val) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= nq) return;
    for (int64_t s = seg_off[i], e = s + nseg[i]; s < e; ++s) {
        seg_q[s] = static_cast<int32_t>(i);
        key[s] = static_cast<uint32_t>(seg_list[s]);
        val[s] = static_cast<int32_t>(s);
    }
}

__global__ void seg_hist_kernel(const uint32_t *__restrict__ skey, int64_t total, int32_t *__restrict__ cnt) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t < total) atomicAdd(&cnt[skey[t]], 1);
}

// items of list p: its segments (sorted positions [start[p], start[p] + cnt[p])) in chunks of qb;
// each item scans the list's rows up to the largest cutoff among its segments
__global__ void seg_items_kernel(const int32_t *__restrict__ cnt, const int32_t *__restrict__ start,
                                 const int32_t *__restrict__ istart, int64_t nr, const int64_t *__restrict__ offsets,
                                 const int32_t *__restrict__ sval, const int32_t *__restrict__ seg_len, int qb,
                                 ScanItem *__restrict__ items, int32_t *__restrict__ nitems) {
    const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (p >= nr) return;
    const int c = cnt[p];
    const int nc = (c + qb - 1) / qb;
    for (int j = 0; j < nc; ++j) {
        ScanItem it;
        it.qbeg = start[p] + j * qb;
        it.qcnt = min(qb, c - j * qb);
        int m = 0;
        for (int e = 0; e < it.qcnt; ++e) m = max(m, seg_len[sval[it.qbeg + e]]);
        it.pbeg = static_cast<int32_t>(offsets[p]);
        it.pcnt = m;
        items[istart[p] + j] = it;
    }
    if (p == nr - 1) *nitems = istart[p] + nc;
}

// positions in list order: query, cutoff, output row, and the initial bound from the query's
// gamma_k (the k nearest representatives are points of X, so the k-th neighbour lies within
// gamma_k: S <= gamma^p fac, as in select.cu, keeps every possible member of the answer)
__global__ void seg_positions_kernel(const int32_t *__restrict__ sval, int64_t total, const int32_t *__restrict__ seg_q,
                                     const int32_t *__restrict__ seg_len, const float *__restrict__ gamma, int d,
                                     int metric, int32_t *__restrict__ qorder, int32_t *__restrict__ qcut,
                                     int64_t *__restrict__ qout, float *__restrict__ qthr) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t >= total) return;
    const int32_t s = sval[t];
    const int32_t qi = seg_q[s];
    qorder[t] = qi;
    qcut[t] = seg_len[s];
    qout[t] = s;
    const float g = gamma[qi];
    const float fac = 1.0f + static_cast<float>(4 * d + 16) * (1.0f / 16777216.0f);
    const float gp = metric == RBC_L2 ? g * g * (1.0f + 1.0f / 8388608.0f) : g;
    qthr[t] = fmaf(gp, fac, static_cast<float>(d) * 1e-35f);
}

// per query: the k smallest keys over its segments' k-key rows (ascending; empty = ~0)
template <int KT>
__global__ void seg_merge_kernel(const uint64_t *__restrict__ seg_keys, const int64_t *__restrict__ seg_off,
                                 const int32_t *__restrict__ nseg, int64_t nq, int k, uint64_t *__restrict__ out) {
    const int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= nq) return;
    uint64_t best[KT];
#pragma unroll
    for (int j = 0; j < KT; ++j) best[j] = kEmptyKey;
    const uint64_t *src = seg_keys + seg_off[i] * k;
    for (int64_t t = lane, e = static_cast<int64_t>(nseg[i]) * k; t < e; t += 32) {
        const uint64_t key = src[t];
        if (key < best[KT - 1]) sorted_insert<KT>(best, key);
    }
    warp_merge_sorted<KT>(best, k, out + i * k);
}

int simt_dmax(int d) { return d <= 24 ? 24 : d <= 64 ? 64 : 128; }
int simt_kt(int k) { return k <= 1 ? 1 : k <= 4 ? 4 : k <= 16 ? 16 : 32; }
// queries per lane: each shared-memory row read serves QPT queries, as registers allow
// (grouped items with small groups use one: a lane slot left empty costs a full scan)
int simt_qpt(int d, int k) { return d <= 64 && k <= 4 ? 2 : 1; }  // (k > 4: the k-best registers spill at two)
// grouped items: enough queries per lane that one chunk holds a typical group (every chunk of a
// group scans the whole s-list, so an almost empty second chunk costs as much as a full one)
int simt_qpt_grouped(int d, int k, int64_t nq, int64_t nr) {
    const int64_t mean = (nq + nr - 1) / (nr > 0 ? nr : 1);
    // (three queries per lane for ~69-query groups measured slower at cfg4: 1.26 vs 1.06 ms)
    return d <= 64 && k <= 4 && mean > 96 ? 2 : 1;
}
int simt_tp(int d4) { return d4 <= 32 ? 128 : 64; }

size_t simt_smem(int d4, int k, int qpt) {
    const int tp = simt_tp(d4);
    const size_t tiles = 2 * static_cast<size_t>(tp) * d4 * sizeof(float);
    const size_t merge = static_cast<size_t>(kW) * 32 * qpt * k * sizeof(uint64_t);
    return (tiles > merge ? tiles : merge) + kW * 32 * qpt * sizeof(float) + kQLen * kT * 2 * sizeof(float);
}

template <int METRIC, int DMAX, int KT, int QPT>
int launch_kt(const SimtSegParams &P, unsigned grid, cudaStream_t st) {
    const size_t smem = simt_smem(P.d4, P.k, QPT);
    if (P.qcut) {  // segment items: exact L1 stage 2 only (L2 stage 2 runs on the tensor cores)
        if constexpr (METRIC == RBC_L1 && QPT == 1) {
            auto *fn = simt_seg_kernel<METRIC, DMAX, KT, QPT>;
            if (smem > 48 * 1024)
                RBC_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
            fn<<<grid, kT, smem, st>>>(P);
            RBC_LAUNCHED();
            return RBC_OK;
        }
        return fail(RBC_EINVAL, "simt segment scan: L1, one query per lane");
    }
    auto *fn = simt_tile_kernel<METRIC, DMAX, KT, QPT>;
    if (smem > 48 * 1024)
        RBC_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    fn<<<grid, kT, smem, st>>>(static_cast<const SimtParams &>(P));
    RBC_LAUNCHED();
    return RBC_OK;
}

template <int METRIC, int DMAX, int QPT>
int launch_qpt(const SimtSegParams &P, unsigned grid, cudaStream_t st) {
    switch (simt_kt(P.k)) {
        case 1: return launch_kt<METRIC, DMAX, 1, QPT>(P, grid, st);
        case 4: return launch_kt<METRIC, DMAX, 4, QPT>(P, grid, st);
        default: return launch_kt<METRIC, DMAX, 16, QPT>(P, grid, st);
    }
}

template <int METRIC, int DMAX>
int launch_dmax(const SimtSegParams &P, unsigned grid, cudaStream_t st) {
    if (P.k > 16) return launch_kt<METRIC, DMAX, 32, 1>(P, grid, st);
    if constexpr (DMAX <= 64) {
        if (P.qpt == 2) {  // k <= 4
            if (simt_kt(P.k) == 1) return launch_kt<METRIC, DMAX, 1, 2>(P, grid, st);
            return launch_kt<METRIC, DMAX, 4, 2>(P, grid, st);
        }
    }
    return launch_qpt<METRIC, DMAX, 1>(P, grid, st);
}

template <int METRIC>
int launch_metric(const SimtSegParams &P, unsigned grid, cudaStream_t st) {
    switch (simt_dmax(P.d)) {
        case 24: return launch_dmax<METRIC, 24>(P, grid, st);
        case 64: return launch_dmax<METRIC, 64>(P, grid, st);
        default: return launch_dmax<METRIC, 128>(P, grid, st);
    }
}

std::atomic<int64_t> g_simt_calls{0};

int simt_launch(SimtSegParams P, int metric, int64_t grid, cudaStream_t st) {
    g_simt_calls.fetch_add(1);
    if (grid > 0x7FFFFFFF) return fail(RBC_EINVAL, "simt scan: too many queries for one call");
    P.d4 = (P.d + 3) & ~3;
    P.tp = simt_tp(P.d4);
    return metric == RBC_L2 ? launch_metric<RBC_L2>(P, static_cast<unsigned>(grid), st)
                            : launch_metric<RBC_L1>(P, static_cast<unsigned>(grid), st);
}

}  // namespace

bool simt_supported(int d, int k) { return d >= 1 && d <= 128 && k >= 1 && k <= 32; }

bool simt_one_shot_supported(const rbc_index *idx, int64_t nq, int k) {
    return idx->kind == 1 && idx->x4 != nullptr && simt_supported(idx->d, k) && k <= idx->s &&
           nq < (int64_t(1) << 31) && idx->nr * static_cast<int64_t>(idx->s) < (int64_t(1) << 31) &&
           idx->s < (1 << 28) &&
           nq * idx->s >= simt_min_pairs();
}

int simt_pad_rows(const float *src, const int32_t *ids, int64_t rows, int d, float *dst, cudaStream_t st) {
    if (rows == 0) return RBC_OK;
    const int d4 = (d + 3) & ~3;
    pad_rows_kernel<<<grid_for(rows * d4, 256, 148 * 64), 256, 0, st>>>(src, ids, rows, d, d4, dst);
    RBC_LAUNCHED();
    return RBC_OK;
}

// k nearest keys (ascending) of every q row over the rows of x; ids = row index (pid
// nullptr) or pid[row].  x4: x with the padded stride, when the caller has it.
int simt_dense_topk(const float *q, int64_t nq, const float *x, int64_t n, int d, int metric, int k,
                    const int32_t *pid, uint64_t *keys, cudaStream_t st, const float *x4) {
    if (nq == 0) return RBC_OK;
    if (!simt_supported(d, k)) return fail(RBC_EINVAL, "simt scan: unsupported d or k");
    if (n >= (int64_t(1) << 31)) return fail(RBC_EINVAL, "simt scan: too many points for one call");
    const int d4 = (d + 3) & ~3;
    DevBuf<float> padded;
    if (!x4) {
        if (d4 == d && (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
            x4 = x;
        } else {
            RBC_CHECK(padded.alloc(n * d4, st));
            RBC_CHECK(simt_pad_rows(x, nullptr, n, d, padded.get(), st));
            x4 = padded.get();
        }
    }
    // query chunks of 32 QPT x point splits: splits (merged by merge_parts) only when the
    // chunks alone leave the GPU short of ~4 CTAs per SM, each split >= 4 tiles
    const int qpt = simt_qpt(d, k);
    const int qb = 32 * qpt;
    const int64_t nqc = (nq + qb - 1) / qb;
    int64_t splits = (148 * 4 + nqc - 1) / nqc;
    const int64_t max_splits = (n + 4 * simt_tp(d4) - 1) / (4 * simt_tp(d4));
    if (splits > max_splits) splits = max_splits;
    if (splits < 1) splits = 1;
    if (splits < (n >> 27) + 1) splits = (n >> 27) + 1;  // rows of a split < 2^28 (queue encoding)
    const int64_t pchunk = (n + splits - 1) / splits;
    splits = (n + pchunk - 1) / pchunk;
    DevBuf<uint64_t> part;
    if (splits > 1) RBC_CHECK(part.alloc(splits * nq * k, st));
    SimtSegParams P{};
    P.q = q;
    P.nq = nq;
    P.d = d;
    P.d4 = d4;
    P.p = x4;
    P.pid = pid;
    P.nqc = nqc;
    P.np = n;
    P.pchunk = pchunk;
    P.k = k;
    P.qpt = qpt;
    P.out = splits > 1 ? part.get() : keys;
    RBC_CHECK(simt_launch(P, metric, nqc * splits, st));
    if (splits > 1) RBC_CHECK(merge_parts(part.get(), static_cast<int>(splits), nq, k, k, keys, st));
    return RBC_OK;
}

// one-shot list scan: query i scans the s-list of its nearest representative key_id(near[i])
// (rows [r s, r s + s) of idx->x4, ids idx->lists)
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
    const int qpt = simt_qpt_grouped(idx->d, k, nq, idx->nr);
    const int qb = 32 * qpt;
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
    SimtSegParams P{};
    P.q = q;
    P.nq = nq;
    P.d = idx->d;
    P.qorder = qorder.get();
    P.items = items.get();
    P.nitems = nitems.get();
    P.p = idx->x4;
    P.pid = idx->lists;
    P.k = k;
    P.qpt = qpt;
    P.out = keys;
    return simt_launch(P, idx->metric, max_items, st);
}

bool simt_exact_supported(const rbc_index *idx, int64_t nq, int k) {
    // (a list's rows are encoded in 28 bits in the candidate queues: n_local < 2^28 bounds every list)
    return idx->kind == 0 && idx->metric == RBC_L1 && idx->x4 != nullptr && simt_supported(idx->d, k) && idx->n_local < (int64_t(1) << 28) &&
           nq < (int64_t(1) << 31) && nq * idx->nr >= simt_min_pairs();
}

// Exact-search stage 2 (search.py:183-186) on the SIMT filter: every query's surviving segments
// (list p, cutoff) regrouped by list -- one item per (list, chunk of its segments) scanning the
// list's rows up to the chunk's largest cutoff, each position stopping at its own -- then the
// per-segment k-key rows merged per query.
int simt_exact_stage2(const rbc_index *idx, const float *q, int64_t nq, int k, const int64_t *seg_off,
                      const int32_t *nseg, const int32_t *seg_list, const int32_t *seg_len, const float *gamma,
                      int64_t total, uint64_t *keys, cudaStream_t st) {
    if (nq == 0) return RBC_OK;
    if (total >= (int64_t(1) << 31)) return fail(RBC_EINVAL, "simt stage 2: too many segments");
    const int64_t nr = idx->nr;
    const int64_t T = total > 0 ? total : 1;
    DevBuf<int32_t> seg_q, val, sval, cnt, start, nchunk, istart, nitems, qorder, qcut;
    DevBuf<float> qthr;
    DevBuf<uint32_t> key, skey;
    DevBuf<int64_t> qout;
    DevBuf<ScanItem> items;
    DevBuf<uint64_t> seg_keys;
    RBC_CHECK(seg_q.alloc(T, st));
    RBC_CHECK(key.alloc(T, st));
    RBC_CHECK(skey.alloc(T, st));
    RBC_CHECK(val.alloc(T, st));
    RBC_CHECK(sval.alloc(T, st));
    RBC_CHECK(cnt.alloc(nr, st));
    RBC_CHECK(start.alloc(nr, st));
    RBC_CHECK(nchunk.alloc(nr, st));
    RBC_CHECK(istart.alloc(nr, st));
    RBC_CHECK(nitems.alloc(1, st));
    RBC_CHECK(qorder.alloc(T, st));
    RBC_CHECK(qcut.alloc(T, st));
    RBC_CHECK(qout.alloc(T, st));
    RBC_CHECK(qthr.alloc(T, st));
    RBC_CHECK(seg_keys.alloc(T * k, st));
    seg_query_kernel<<<grid_for(nq, 256), 256, 0, st>>>(seg_off, nseg, nq, seg_list, seg_q.get(), key.get(), val.get());
    RBC_LAUNCHED();
    int kb = 1;
    while ((int64_t(1) << kb) < nr) ++kb;
    size_t tb = 0, tb2 = 0, tb3 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, key.get(), skey.get(), val.get(), sval.get(), total, 0, kb, st);
    cub::DeviceScan::ExclusiveSum(nullptr, tb2, cnt.get(), start.get(), nr, st);
    cub::DeviceScan::ExclusiveSum(nullptr, tb3, nchunk.get(), istart.get(), nr, st);
    DevBuf<unsigned char> tmp;
    RBC_CHECK(tmp.alloc(std::max(tb, std::max(tb2, tb3)), st));
    if (total > 0) {
        RBC_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, key.get(), skey.get(), val.get(), sval.get(), total, 0,
                                                 kb, st));
        note_launch();
    }
    const int qpt = 1;  // (simt_seg_kernel: one segment per lane)
    const int qb = 32 * qpt;
    RBC_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(int32_t) * nr, st));
    seg_hist_kernel<<<grid_for(T, 256), 256, 0, st>>>(skey.get(), total, cnt.get());
    RBC_LAUNCHED();
    near_chunks_kernel<<<grid_for(nr, 256), 256, 0, st>>>(cnt.get(), nr, qb, nchunk.get());
    RBC_LAUNCHED();
    RBC_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb2, cnt.get(), start.get(), nr, st));
    RBC_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb3, nchunk.get(), istart.get(), nr, st));
    note_launch(2);
    const int64_t max_items = std::min<int64_t>(nr, T) + T / qb + 1;
    RBC_CHECK(items.alloc(max_items, st));
    seg_items_kernel<<<grid_for(nr, 256), 256, 0, st>>>(cnt.get(), start.get(), istart.get(), nr, idx->offsets,
                                                       sval.get(), seg_len, qb, items.get(), nitems.get());
    RBC_LAUNCHED();
    seg_positions_kernel<<<grid_for(T, 256), 256, 0, st>>>(sval.get(), total, seg_q.get(), seg_len, gamma, idx->d,
                                                          idx->metric, qorder.get(), qcut.get(), qout.get(), qthr.get());
    RBC_LAUNCHED();
    SimtSegParams P{};
    P.q = q;
    P.nq = T;
    P.d = idx->d;
    P.qorder = qorder.get();
    P.items = items.get();
    P.nitems = nitems.get();
    P.p = idx->x4;
    P.pid = idx->perm;
    P.qcut = qcut.get();
    P.qout = qout.get();
    P.qthr = qthr.get();
    P.k = k;
    P.qpt = qpt;
    P.out = seg_keys.get();
    if (total > 0) RBC_CHECK(simt_launch(P, idx->metric, max_items, st));
    const unsigned mgrid = grid_for(nq * 32, 256);
    const int kt = simt_kt(k);
    if (kt == 1) seg_merge_kernel<1><<<mgrid, 256, 0, st>>>(seg_keys.get(), seg_off, nseg, nq, k, keys);
    else if (kt == 4) seg_merge_kernel<4><<<mgrid, 256, 0, st>>>(seg_keys.get(), seg_off, nseg, nq, k, keys);
    else if (kt == 16) seg_merge_kernel<16><<<mgrid, 256, 0, st>>>(seg_keys.get(), seg_off, nseg, nq, k, keys);
    else seg_merge_kernel<32><<<mgrid, 256, 0, st>>>(seg_keys.get(), seg_off, nseg, nq, k, keys);
    RBC_LAUNCHED();
    return RBC_OK;
}

// padded SIMT operands of an index: the representatives (both kinds) and, one-shot, the
// s-lists' rows gathered per list; exact L1 indexes: the list-ordered rows (stage 2)
int simt_index_prepare(rbc_index *idx, cudaStream_t st) {
    if (idx->d > 128 || (idx->kind == 0 && idx->metric != RBC_L1)) return RBC_OK;
    const int d4 = (idx->d + 3) & ~3;
    if (cudaMalloc(&idx->reps4, sizeof(float) * idx->nr * d4) != cudaSuccess)
        return fail(RBC_ENOMEM, "simt operands (representatives)");
    idx->bytes += sizeof(float) * idx->nr * d4;
    RBC_CHECK(simt_pad_rows(idx->reps, nullptr, idx->nr, idx->d, idx->reps4, st));
    if (idx->kind == 0) {
        // exact indexes: L1 only (L2 stage 2 runs on the tensor cores)
        if (idx->metric != RBC_L1 || idx->n_local == 0 || idx->n_local >= (int64_t(1) << 31)) return RBC_OK;
        if (cudaMalloc(&idx->x4, sizeof(float) * idx->n_local * d4) != cudaSuccess)
            return fail(RBC_ENOMEM, "simt operands (list-ordered rows)");
        idx->bytes += sizeof(float) * idx->n_local * d4;
        RBC_CHECK(simt_pad_rows(idx->xp, nullptr, idx->n_local, idx->d, idx->x4, st));
    } else {
        const int64_t rows = idx->nr * static_cast<int64_t>(idx->s);
        if (rows >= (int64_t(1) << 31)) return RBC_OK;
        if (cudaMalloc(&idx->x4, sizeof(float) * rows * d4) != cudaSuccess)
            return fail(RBC_ENOMEM, "simt operands (list rows)");
        idx->bytes += sizeof(float) * rows * d4;
        RBC_CHECK(simt_pad_rows(idx->x, idx->lists, rows, idx->d, idx->x4, st));
    }
    return RBC_OK;
}

}  // namespace rbc

extern "C" int64_t rbc_simt_scan_calls(void) { return rbc::g_simt_calls.load(); }
