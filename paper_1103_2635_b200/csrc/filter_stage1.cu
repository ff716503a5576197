// filter_stage1.cu -- exact-search stage 1 + pruning for the indexes the tensor-core stage 1
// (tc_stage1.cu: L2, d <= 64) does not cover: d > 64 (cfg5, d = 128) and L1.
//
// The reference computes every dist(q, r) exactly (search.py:178), takes the k-th smallest
// as gamma_k (:181), keeps r iff  d <= 3 gamma and (d < gamma + psi_r or d <= gamma)
// (:62-74), counts the two pruning tests (:194-195) and scans each survivor's list up to
// 4 gamma (:77-82, 183-186).  Computing the whole |Q| x |R| block in fp64 is fp64-issue
// bound (d = 128: ~1.2 ms per 10k queries x 4k reps).  Here:
//
//   filter  S~ = fp32 SIMT sum of the per-coordinate terms for every (q, r) (packed FADD2 /
//           FFMA2, 64 x 128 register-tiled block).  All terms are non-negative, so
//           |S~ - S| <= (4d + 16) 2^-24 S + d 1e-35 (the SIMT filter's bound, simt_scan.cu)
//           and the exact f32 distance lies in [lo(S~), hi(S~)] (directed roundings).
//   count   one warp per query.  The k smallest S~ bound gamma_k from above, so every rep
//           whose lower bound reaches that is a gamma candidate: their exact distances give gamma_k and the
//           nearest rep.  Then every rep is classified with the reference's predicates at
//           both ends of its interval -- survives() falls and both pruning tests rise
//           monotonically with the distance, so equal answers at lo and hi decide the rep.
//           Only undecided reps and survivors get the exact fp64 distance (exact_dist, the
//           reference arithmetic), 32 at a time (one per lane), and the survivors' 4 gamma
//           cutoffs are binary searches run 32 at a time as well (the old per-rep loop
//           serialised one search's dependent loads per iteration).
//           All of it compares S~ against thresholds mapped into the S domain (t^2 for L2),
//           so a rep costs a few FFMA / FSETP; the row is read 4 values per lane at a time.
//           Output: a bit per (query, rep) with a segment, and for those the cutoff length
//           (len[q][r]) and the exact distance, written over the S~ entry.
//   fill    the segment bits -> the segment arrays, ascending rep position (the order
//           prune_fill_warp_kernel emits).
// Every output (gamma, candidates, both pruning counts, the segments) is the exact path's.
// A query with more than kCap gamma candidates (ties or near-ties in the hundreds) sets the
// fail flag and the caller redoes the batch with the exact path (search.cu).
#include <cub/cub.cuh>

#include <atomic>

#include "common.cuh"
#include "index.cuh"
#include "prune_math.cuh"
#include "search.cuh"
#include "tc_scan.cuh"

namespace rbc {

namespace {

// ---- filter: S~ for every (query, rep) -----------------------------------------------
constexpr int kFq = 64;         // queries per block
constexpr int kFr = 128;        // reps per block
constexpr int kFc = 16;         // coordinates per shared-memory stage
constexpr int kQs = 2 * kFq + 4;  // query row stride: each value twice ({q, q} pairs), padded
constexpr int kRs = kFr + 4;

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

// 256 threads: thread (tx, ty) owns queries ty*4 .. +3 and reps tx*4 .. +3, 64 + tx*4 .. +3.
// VEC (d % 4 == 0, 16-byte rows): each stage is one float4 of q and two of r per thread,
// loaded into registers one stage ahead so their latency overlaps the current stage's math.
template <int METRIC, bool VEC>
__global__ void __launch_bounds__(256) s1_filter_kernel(const float *__restrict__ q, int64_t m,
                                                        const float *__restrict__ r, int64_t nr, int d,
                                                        float *__restrict__ S, int64_t ld) {
    __shared__ __align__(16) float qs[kFc][kQs];
    __shared__ __align__(16) float rs[kFc][kRs];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t i0 = static_cast<int64_t>(blockIdx.x) * kFq, j0 = static_cast<int64_t>(blockIdx.y) * kFr;
    float2 acc[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = make_float2(0.f, 0.f);
    // VEC staging: thread t loads coordinates 4 (t & 3) .. +3 of query row t >> 2 and of rep
    // rows t >> 2 and 64 + (t >> 2)
    const int vr = threadIdx.x >> 2, vc = 4 * (threadIdx.x & 3);
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 pq = z4, pa = z4, pb = z4;
    auto vload = [&](int k0) {
        const bool cin = k0 + vc < d;
        pq = cin && i0 + vr < m ? __ldg(reinterpret_cast<const float4 *>(q + (i0 + vr) * d + k0 + vc)) : z4;
        pa = cin && j0 + vr < nr ? __ldg(reinterpret_cast<const float4 *>(r + (j0 + vr) * d + k0 + vc)) : z4;
        pb = cin && j0 + 64 + vr < nr ? __ldg(reinterpret_cast<const float4 *>(r + (j0 + 64 + vr) * d + k0 + vc)) : z4;
    };
    if (VEC) vload(0);
    for (int k0 = 0; k0 < d; k0 += kFc) {
        if (VEC) {
            const float qv4[4] = {pq.x, pq.y, pq.z, pq.w}, av4[4] = {pa.x, pa.y, pa.z, pa.w},
                        bv4[4] = {pb.x, pb.y, pb.z, pb.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                *reinterpret_cast<float2 *>(&qs[vc + j][2 * vr]) = make_float2(qv4[j], qv4[j]);
                rs[vc + j][vr] = av4[j];
                rs[vc + j][64 + vr] = bv4[j];
            }
        } else {
            // stage: coalesced along the coordinates, transposed into [coordinate][row]
            for (int e = threadIdx.x; e < kFq * kFc; e += 256) {
                const int row = e / kFc, c = e % kFc;
                const float v = (i0 + row < m && k0 + c < d) ? q[(i0 + row) * d + k0 + c] : 0.f;
                *reinterpret_cast<float2 *>(&qs[c][2 * row]) = make_float2(v, v);
            }
            for (int e = threadIdx.x; e < kFr * kFc; e += 256) {
                const int row = e / kFc, c = e % kFc;
                rs[c][row] = (j0 + row < nr && k0 + c < d) ? r[(j0 + row) * d + k0 + c] : 0.f;
            }
        }
        __syncthreads();
        if (VEC && k0 + kFc < d) vload(k0 + kFc);
#pragma unroll 4
        for (int c = 0; c < kFc; ++c) {
            const float4 qa = *reinterpret_cast<const float4 *>(&qs[c][8 * ty]);
            const float4 qb = *reinterpret_cast<const float4 *>(&qs[c][8 * ty + 4]);
            const float4 ra = *reinterpret_cast<const float4 *>(&rs[c][4 * tx]);
            const float4 rb = *reinterpret_cast<const float4 *>(&rs[c][64 + 4 * tx]);
            const float2 qv[4] = {make_float2(qa.x, qa.y), make_float2(qa.z, qa.w), make_float2(qb.x, qb.y),
                                  make_float2(qb.z, qb.w)};
            const float2 rv[4] = {make_float2(ra.x, ra.y), make_float2(ra.z, ra.w), make_float2(rb.x, rb.y),
                                  make_float2(rb.z, rb.w)};
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const float2 t = sub2(rv[v], qv[u]);
                    if (METRIC == RBC_L2) {
                        acc[u][v] = fma2(t, t, acc[u][v]);
                    } else {
                        acc[u][v].x += fabsf(t.x);
                        acc[u][v].y += fabsf(t.y);
                    }
                }
        }
        __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int64_t i = i0 + 4 * ty + u;
        if (i >= m) continue;
        float *row = S + i * ld;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int64_t j = j0 + (v < 2 ? 4 * tx + 2 * v : 64 + 4 * tx + 2 * (v - 2));
            if (j < nr) row[j] = acc[u][v].x;
            if (j + 1 < nr) row[j + 1] = acc[u][v].y;
        }
    }
}

// ---- count: gamma_k, predicates, cutoffs --------------------------------------------
constexpr int kWarps = 8;
constexpr int kCap = 256;   // gamma candidates per query (more: fail -> exact path)
constexpr int kWork = 64;   // pending exact evaluations per warp
constexpr int kU = 4;       // row values per lane in flight (128 reps per warp step)

// S (the reference's fp64 sum) lies in [S~ dn - tiny, S~ up + tiny]; up / dn carry the
// filter's relative bound plus 2^-17 of slack for everything rounded after it (the f32
// rounding of the distance and its square root, the fp32 thresholds and these products), so
// every comparison below is decided in plain fp32 and stays conservative.
struct Bounds {
    float up, dn, tiny;
};

struct CountOut {
    float *gamma;
    int32_t *nseg;
    int64_t *cand;
    int32_t *pr, *p3;
    uint64_t *order_key;
    uint32_t *mask;  // [m][nw] bit p: rep p has a segment
    int32_t *fail;
};

// a distance threshold t (fp32 rounding of the reference's fp64 threshold) in the domain of
// S~: t^2 for L2, t for L1.  A positive threshold whose square underflows decides nothing.
template <int METRIC>
__device__ __forceinline__ float sdom(float t, bool &valid) {
    const float t2 = METRIC == RBC_L2 ? t * t : t;
    valid = (t == 0.f || t2 >= 1e-30f) && t2 < __int_as_float(0x7f800000);
    return t2;
}

// (a variant staging each warp's S~ row in shared memory once, 4 warps per block, measured
// slower at cfg5: 476 vs 351 us -- the kernel's time is the latency of the exact distances,
// which then had a third of the warps to hide it)
template <int METRIC, int KT>
__global__ void __launch_bounds__(kWarps * 32, 4) s1_count_kernel(const float *__restrict__ q, int64_t m,
                                                               const float *__restrict__ reps, int64_t nr, int d,
                                                               int k, Bounds bd, const float *__restrict__ radii,
                                                               const int64_t *__restrict__ offsets,
                                                               const float *__restrict__ list_dists,
                                                               float *__restrict__ d1, int32_t *__restrict__ len_out,
                                                               int64_t ld, CountOut out) {
    __shared__ int32_t s_cp[kWarps][kCap];
    __shared__ float s_cd[kWarps][kCap];
    __shared__ int32_t s_work[kWarps][kWork];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * kWarps + w;
    if (i >= m) return;
    const float inf = __int_as_float(0x7f800000);
    float *srow = d1 + i * ld;
    int32_t *lrow = len_out + i * ld;
    const float *rd = srow;
    const float *qi = q + i * d;
    const int64_t nw = (nr + 31) >> 5;
    uint32_t *mrow = out.mask + i * nw;

    // pass 1: the k smallest S~ (S~ -> upper bound is monotone)
    float best[KT];
#pragma unroll
    for (int j = 0; j < KT; ++j) best[j] = inf;
    // thr: the k-th smallest of the 32 lane minima, an upper bound of the row's k-th smallest
    // (k <= 32 lanes each hold a value at or below it), refreshed after 1, 2, 4, ... steps so
    // that late values rarely enter the per-lane lists
    float thr = inf;
    int64_t step = 0;
    for (int64_t p0 = 0; p0 < nr; p0 += 32 * kU) {
        float sv[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int64_t p = p0 + 32 * u + lane;
            sv[u] = p < nr ? rd[p] : inf;
        }
        if (++step > 1 && (step & (step - 1)) == 0) {
            float v = best[0];  // bitonic sort of the lane minima, ascending
#pragma unroll
            for (int size = 2; size <= 32; size <<= 1)
#pragma unroll
                for (int stride = size >> 1; stride > 0; stride >>= 1) {
                    const float o = __shfl_xor_sync(0xffffffffu, v, stride);
                    v = (((lane & stride) == 0) == ((lane & size) == 0)) ? fminf(v, o) : fmaxf(v, o);
                }
            thr = __shfl_sync(0xffffffffu, v, k - 1);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            float x = sv[u];
            if (x < best[KT - 1] && x <= thr) {
#pragma unroll
                for (int j = 0; j < KT; ++j) {
                    const float a = fminf(best[j], x), b = fmaxf(best[j], x);
                    best[j] = a;
                    x = b;
                }
            }
        }
    }
    float Sk = best[0];
    for (int rr = 0; rr < k; ++rr) {
        unsigned long long h = (static_cast<unsigned long long>(__float_as_uint(best[0])) << 32) | lane;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long x = __shfl_xor_sync(0xffffffffu, h, o);
            h = x < h ? x : h;
        }
        Sk = __uint_as_float(static_cast<uint32_t>(h >> 32));
        if (static_cast<int>(h & 31) == lane) {
#pragma unroll
            for (int j = 0; j < KT - 1; ++j) best[j] = best[j + 1];
            best[KT - 1] = inf;
        }
    }
    // those k reps all lie within T2 (S domain), so gamma_k does too; a rep can only be at or
    // below gamma_k if its lower bound reaches T2 (non-finite sums: always a candidate)
    const float T2 = fmaf(Sk, bd.up, bd.tiny);

    // pass 2: gamma candidates, ascending rep position
    int nc = 0;
    for (int64_t p0 = 0; p0 < nr; p0 += 32 * kU) {
        float sv[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int64_t p = p0 + 32 * u + lane;
            sv[u] = p < nr ? rd[p] : 0.f;
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int64_t p = p0 + 32 * u + lane;
            const bool c = p < nr && (!(sv[u] < inf) || !(fmaf(sv[u], bd.dn, -bd.tiny) > T2));
            const unsigned bal = __ballot_sync(0xffffffffu, c);
            const int at = nc + __popc(bal & ((1u << lane) - 1u));
            if (c && at < kCap) s_cp[w][at] = static_cast<int32_t>(p);
            nc += __popc(bal);
        }
    }
    if (nc > kCap) {
        if (lane == 0) atomicExch(out.fail, 1);
        return;
    }
    __syncwarp();
    for (int j = lane; j < nc; j += 32) s_cd[w][j] = exact_dist<METRIC, 8>(qi, reps + static_cast<int64_t>(s_cp[w][j]) * d, d);
    __syncwarp();
    // gamma_k = k-th smallest exact candidate distance; nearest rep = the first (ties: lowest position)
    unsigned removed = 0;  // bit t: entry lane + 32 t taken
    float g32 = 0.f;
    unsigned long long near = ~0ull;
    for (int rr = 0; rr < k; ++rr) {
        unsigned long long h = ~0ull;
        for (int t = 0; lane + 32 * t < nc; ++t) {
            const int j = lane + 32 * t;
            if (removed >> t & 1u) continue;
            const unsigned long long x = (static_cast<unsigned long long>(__float_as_uint(s_cd[w][j])) << 32) | j;
            h = x < h ? x : h;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long x = __shfl_xor_sync(0xffffffffu, h, o);
            h = x < h ? x : h;
        }
        const int j = static_cast<int>(h & 0xFFFFFFFFu);
        if ((j & 31) == lane) removed |= 1u << (j >> 5);
        g32 = __uint_as_float(static_cast<uint32_t>(h >> 32));
        if (rr == 0) near = pack_key(g32, static_cast<uint32_t>(s_cp[w][j]));
    }
    const double g = g32, cut = 4.0 * g;
    // per-query thresholds in the S~ domain: gamma (search.py:195's "d > gamma" side of the radius
    // test, and the d <= gamma survival clause) and 3 gamma
    bool vB, vC;
    const float tB = sdom<METRIC>(g32, vB), tC = sdom<METRIC>(3.0f * g32, vC);

    for (int64_t t = lane; t < nw; t += 32) mrow[t] = 0u;
    __syncwarp();

    // pass 3: classify every rep; exact distances for the undecided and the survivors
    long long cand = 0;
    int nseg = 0, pr = 0, p3 = 0;
    unsigned first = 0xFFFFFFFFu;
    int nw_ = 0;
    auto drain = [&](int cnt) {  // entries 0 .. cnt-1 (cnt <= 32), one per lane
        if (lane < cnt) {
            const int32_t p = s_work[w][lane];
            const float dist = exact_dist<METRIC, 8>(qi, reps + static_cast<int64_t>(p) * d, d);
            const float rad = radii[p];
            pr += pruned_radius(dist, rad, g) ? 1 : 0;
            p3 += pruned_3gamma(dist, g) ? 1 : 0;
            if (survives(dist, rad, g)) {
                const int32_t len =
                    list_cutoff_dev(list_dists + offsets[p], static_cast<int32_t>(offsets[p + 1] - offsets[p]), cut);
                cand += len;
                if (len > 0) {
                    ++nseg;
                    first = min(first, static_cast<unsigned>(p));
                    srow[p] = dist;
                    lrow[p] = len;
                    atomicOr(mrow + (p >> 5), 1u << (p & 31));
                }
            }
        }
    };
    for (int64_t p0 = 0; p0 < nr; p0 += 32 * kU) {
        float sv[kU], rv[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int64_t p = p0 + 32 * u + lane;
            sv[u] = p < nr ? rd[p] : 0.f;
            rv[u] = p < nr ? radii[p] : 0.f;
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int64_t p = p0 + 32 * u + lane;
            bool need = false;
            if (p < nr) {
                const float s = sv[u];
                need = true;
                if (s < inf) {
                    const float sH = fmaf(s, bd.up, bd.tiny), sL = fmaf(s, bd.dn, -bd.tiny);
                    bool vA;
                    const float tA = sdom<METRIC>(g32 + rv[u], vA);
                    const bool ltA = vA && sH < tA, gtA = vA && sL > tA;
                    const bool ltB = vB && sH < tB, gtB = vB && sL > tB;
                    const bool ltC = vC && sH < tC, gtC = vC && sL > tC;
                    // pruned by radius: d >= gamma + psi and d > gamma (search.py:194)
                    const bool pr_t = gtA && gtB, pr_f = ltA || ltB;
                    // survives: d <= 3 gamma and (d < gamma + psi or d <= gamma) (search.py:62-74)
                    const bool sv_f = gtC || (gtA && gtB);
                    need = !(pr_t || pr_f) || !(gtC || ltC) || !sv_f;
                    if (!need) {
                        pr += pr_t ? 1 : 0;
                        p3 += gtC ? 1 : 0;
                    }
                }
            }
            const unsigned bal = __ballot_sync(0xffffffffu, need);
            if (need) s_work[w][nw_ + __popc(bal & ((1u << lane) - 1u))] = static_cast<int32_t>(p);
            nw_ += __popc(bal);
            if (nw_ >= 32) {
                __syncwarp();
                drain(32);
                __syncwarp();
                if (lane < nw_ - 32) s_work[w][lane] = s_work[w][32 + lane];
                nw_ -= 32;
                __syncwarp();
            }
        }
    }
    __syncwarp();
    drain(nw_);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        cand += __shfl_xor_sync(0xffffffffu, cand, o);
        nseg += __shfl_xor_sync(0xffffffffu, nseg, o);
        pr += __shfl_xor_sync(0xffffffffu, pr, o);
        p3 += __shfl_xor_sync(0xffffffffu, p3, o);
        first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
    }
    if (lane == 0) {
        out.gamma[i] = g32;
        out.nseg[i] = nseg;
        out.cand[i] = cand;
        if (out.pr) out.pr[i] = pr;
        if (out.p3) out.p3[i] = p3;
        out.order_key[i] = (static_cast<uint64_t>(first & 0xFFFFFFu) << 24) | (key_id(near) & 0xFFFFFFu);
    }
}

// ---- fill: segment bits -> segments, ascending rep position -------------------------
__global__ void __launch_bounds__(256) s1_fill_kernel(const uint32_t *__restrict__ mask, const int32_t *__restrict__ len,
                                                      const float *__restrict__ d1, int64_t m, int64_t nr,
                                                      int64_t ld, const int64_t *__restrict__ offsets,
                                                      const int64_t *__restrict__ seg_off,
                                                      int64_t *__restrict__ seg_start, int32_t *__restrict__ seg_len,
                                                      int32_t *__restrict__ seg_list, float *__restrict__ seg_d1) {
    const int lane = threadIdx.x & 31;
    const int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    if (i >= m) return;
    const int64_t nw = (nr + 31) >> 5;
    const uint32_t *mrow = mask + i * nw;
    int64_t base = seg_off[i];
    for (int64_t t0 = 0; t0 < nw; t0 += 32) {
        uint32_t bits = t0 + lane < nw ? mrow[t0 + lane] : 0u;
        const int c = __popc(bits);
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        int64_t at = base + incl - c;
        while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            const int64_t p = ((t0 + lane) << 5) + b;
            seg_start[at] = offsets[p];
            seg_len[at] = len[i * ld + p];
            seg_list[at] = static_cast<int32_t>(p);
            seg_d1[at] = d1[i * ld + p];
            ++at;
        }
        base += __shfl_sync(0xffffffffu, incl, 31);
    }
}

std::atomic<int64_t> g_calls{0}, g_fallbacks{0};

struct ToI64 {
    __host__ __device__ int64_t operator()(int32_t v) const { return v; }
};

}  // namespace

int64_t filter_stage1_stride(int64_t nr) { return (nr + 3) & ~int64_t(3); }

bool filter_stage1_supported(const rbc_index *idx, int k) {
    return !force_exact_engine() && k >= 1 && k <= 16 && idx->nr >= k && idx->nr <= int64_t(65535) * kFr &&
           (idx->metric == RBC_L2 || idx->metric == RBC_L1);
}

int filter_stage1(const rbc_index *idx, const float *q, int64_t m, int k, float *d1, int32_t *len, PruneOut &out,
                  bool &ok, cudaStream_t st) {
    ok = false;
    g_calls.fetch_add(1);
    const int64_t nr = idx->nr;
    const int64_t ld = filter_stage1_stride(nr);
    const int d = idx->d;
    RBC_CHECK(out.gamma.alloc(m, st));
    RBC_CHECK(out.nseg.alloc(m, st));
    RBC_CHECK(out.cand.alloc(m, st));
    RBC_CHECK(out.seg_off.alloc(m + 1, st));
    RBC_CHECK(out.order_key.alloc(m, st));
    out.d1 = d1;
    DevBuf<int32_t> flag;
    RBC_CHECK(flag.alloc(1, st));
    RBC_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int32_t), st));
    {
        const dim3 grid(grid_for(m, kFq, 0x7FFFFFFF), grid_for(nr, kFr, 65535));  // nr <= 65535 * kFr (supported)
        const bool vec = (d & 3) == 0 && ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(idx->reps)) & 15) == 0;
        if (idx->metric == RBC_L2) {
            if (vec) s1_filter_kernel<RBC_L2, true><<<grid, 256, 0, st>>>(q, m, idx->reps, nr, d, d1, ld);
            else s1_filter_kernel<RBC_L2, false><<<grid, 256, 0, st>>>(q, m, idx->reps, nr, d, d1, ld);
        } else {
            if (vec) s1_filter_kernel<RBC_L1, true><<<grid, 256, 0, st>>>(q, m, idx->reps, nr, d, d1, ld);
            else s1_filter_kernel<RBC_L1, false><<<grid, 256, 0, st>>>(q, m, idx->reps, nr, d, d1, ld);
        }
        RBC_LAUNCHED();
    }
    // S in [S~ dn - tiny, S~ up + tiny]: the SIMT filter's relative bound (4d + 16) 2^-24 plus
    // 2^-17 of slack (struct Bounds)
    const double e = (4.0 * d + 16.0) / 16777216.0 + 1.0 / 131072.0;
    Bounds bd;
    bd.up = nextafterf(static_cast<float>(1.0 + e), 2.f);
    bd.dn = nextafterf(static_cast<float>(1.0 - e), 0.f);
    bd.tiny = static_cast<float>(d) * 1e-35f;
    DevBuf<uint32_t> mask;
    RBC_CHECK(mask.alloc(m * ((nr + 31) >> 5), st));
    CountOut co{out.gamma.get(), out.nseg.get(), out.cand.get(), out.pr, out.p3, out.order_key.get(), mask.get(),
                flag.get()};
#define RBC_S1_COUNT(M, KT)                                                                                          \
    s1_count_kernel<M, KT><<<grid_for(m, kWarps), kWarps * 32, 0, st>>>(q, m, idx->reps, nr, d, k, bd, idx->radii,  \
                                                                       idx->offsets, idx->list_dists, d1, len, ld,  \
                                                                       co)
    if (idx->metric == RBC_L2) {
        if (k == 1) RBC_S1_COUNT(RBC_L2, 1);
        else if (k <= 4) RBC_S1_COUNT(RBC_L2, 4);
        else RBC_S1_COUNT(RBC_L2, 16);
    } else {
        if (k == 1) RBC_S1_COUNT(RBC_L1, 1);
        else if (k <= 4) RBC_S1_COUNT(RBC_L1, 4);
        else RBC_S1_COUNT(RBC_L1, 16);
    }
#undef RBC_S1_COUNT
    RBC_LAUNCHED();
    RBC_CUDA(cudaMemsetAsync(out.seg_off.get(), 0, sizeof(int64_t), st));
    size_t tb = 0;
    cub::TransformInputIterator<int64_t, ToI64, const int32_t *> in(out.nseg.get(), ToI64());
    cub::DeviceScan::InclusiveSum(nullptr, tb, in, out.seg_off.get() + 1, m, st);
    DevBuf<unsigned char> tmp;
    RBC_CHECK(tmp.alloc(tb, st));
    RBC_CUDA(cub::DeviceScan::InclusiveSum(tmp.get(), tb, in, out.seg_off.get() + 1, m, st));
    note_launch();
    int64_t total = 0;
    int32_t failed = 0;
    RBC_CUDA(cudaMemcpyAsync(&total, out.seg_off.get() + m, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    RBC_CUDA(cudaMemcpyAsync(&failed, flag.get(), sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    RBC_CUDA(cudaStreamSynchronize(st));
    if (failed) {
        g_fallbacks.fetch_add(1);
        return RBC_OK;  // some query had too many gamma candidates: the caller runs the exact path
    }
    out.total_segs = total;
    RBC_CHECK(out.seg_start.alloc(total, st));
    RBC_CHECK(out.seg_len.alloc(total, st));
    RBC_CHECK(out.seg_list.alloc(total, st));
    RBC_CHECK(out.seg_d1.alloc(total, st));
    s1_fill_kernel<<<grid_for(m * 32, 256), 256, 0, st>>>(mask.get(), len, d1, m, nr, ld, idx->offsets, out.seg_off.get(),
                                                          out.seg_start.get(), out.seg_len.get(), out.seg_list.get(),
                                                          out.seg_d1.get());
    RBC_LAUNCHED();
    ok = true;
    return RBC_OK;
}

}  // namespace rbc

extern "C" int64_t rbc_filter_stage1_calls(void) { return rbc::g_calls.load(); }
extern "C" int64_t rbc_filter_stage1_fallbacks(void) { return rbc::g_fallbacks.load(); }
