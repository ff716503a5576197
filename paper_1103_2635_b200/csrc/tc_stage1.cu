// tc_stage1.cu -- exact-search stage 1 (query x representative distances),
// gamma_k and the triangle-inequality pruning, fused on the tensor cores.
//
// The reference computes every dist(q, r) exactly (search.py:178), takes the
// k-th smallest as gamma_k (:181), and keeps r iff
//   d <= 3 gamma  and  (d < gamma + psi_r  or  d <= gamma)      (:62-74)
// counting the two pruning tests (:194-195).  Here each 128-query tile is
// multiplied against all representatives with tcgen05.mma.  Operands are
// centred on the representatives' mean c and split into f16 hi + lo parts
// (three MMAs: hi.hi + hi.lo + lo.hi, ~2^-20 relative precision); the
// per-rep term |r - c|^2 / 2 is folded into the MMA as in tc_stage2.cu.  Every
// d^2 is thereby known inside a rigorous interval [lb, ub]:
//   pass 1: the k smallest upper bounds give a bound U_k; every rep with
//           lb <= U_k is evaluated exactly (fp64, reference arithmetic), so
//           gamma_k and the nearest rep are exact;
//   pass 2: every rep is classified against 3 gamma, gamma and gamma + psi_r
//           with its interval; reps whose class is certain (almost all: far
//           away) are only counted, the rest -- possible survivors and
//           interval straddles -- are recorded for the fix-up kernel, which
//           decides them with exact distances, computes the 4 gamma cutoff by
//           binary search and emits the surviving segments.
// No |Q| x |R| distance matrix is materialised.  Any row that exhausts a
// buffer raises a flag and the caller recomputes the batch with the exact
// path (search.cu), so the result is always the reference's.
#include <cub/cub.cuh>

#include <vector>

#include "common.cuh"
#include "index.cuh"
#include "kernels.cuh"
#include "prune_math.cuh"
#include "search.cuh"
#include "sm100.cuh"
#include "tc_scan.cuh"

namespace rbc {

namespace {

constexpr int kRows = 128;
constexpr int kN = 128;       // representatives per chunk (UMMA N)
constexpr int kStages = 3;
constexpr int kThreads = 192;  // producer, MMA, 4 epilogue warps
constexpr int kP0 = 128, kP1 = 32;
// per row: hi plane (SW128) | lo plane (SW128) | aug plane (SW32, d > 62 only)
constexpr int kStageBytes = kN * (2 * kP0 + kP1);
constexpr int kABytes = kRows * (2 * kP0 + kP1);
constexpr int kMaxRepsSmem = 6144;  // radii staged in shared memory

// hi/lo split: per-product error 3 * 2^-22, fp32 accumulation of <= 208 terms; factor-2 safety, x2 for d^2
constexpr float kC1 = 4.0f * (3.0f / 4194304.0f + 208.0f / 8388608.0f);
constexpr float kC2 = 1.0f / 1048576.0f;
constexpr float kC4 = 1.0f / 1073741824.0f;  // subnormal flush of the lo parts (absolute, scaled)
constexpr float kUp = 1.0f + 1.0f / 1048576.0f;
constexpr float kTie = 1.0f + 1.0f / 524288.0f;
constexpr float kEps = 1.0f / 262144.0f;  // relative slack of the interval classification

struct Tc1Index {
    int64_t nrpad = 0;
    bool plane1 = false;
    uint8_t *rb = nullptr;   // [nrpad] rows of (hi 128 B | lo 128 B | aug 32 B), pre-swizzled
    float *c64 = nullptr;    // [64] centre (mean of the reps), zero padded
    float *stat = nullptr;   // [2] sG, rmax (max |r - c|, rounded up)
    float *psimax = nullptr; // [nchunks] largest list radius of each rep chunk
    float *lskip = nullptr;  // [nr][32] list_dists at the end of each of 32 equal blocks (cutoff skip table)
    float sG = 1.f, rmax = 0.f;
};

// skip table: sample i of list p = list_dists at position min(len, (i+1) * s) - 1, s = ceil(len / 32)
__global__ void list_skip_kernel(const int64_t *__restrict__ offsets, const float *__restrict__ list_dists, int64_t nr,
                                 float *__restrict__ lskip) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t >= nr * 32) return;
    const int64_t p = t >> 5, i = t & 31;
    const int64_t len = offsets[p + 1] - offsets[p];
    const int64_t s = (len + 31) / 32;
    const int64_t pos = min(len, (i + 1) * s) - 1;
    lskip[t] = (len > 0 && pos >= 0) ? list_dists[offsets[p] + pos] : __int_as_float(0x7f800000);
}

// list_cutoff (search.py:77-82) through the skip table: #entries <= thr, f64 compares
__device__ __forceinline__ int32_t list_cutoff_skip(const float *__restrict__ l, int32_t len,
                                                    const float *__restrict__ skip, double thr) {
    if (len == 0) return 0;
    const int32_t s = (len + 31) / 32;
    const float4 *s4 = reinterpret_cast<const float4 *>(skip);
    int b = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const float4 v = __ldg(s4 + c);
        b += (static_cast<double>(v.x) <= thr) + (static_cast<double>(v.y) <= thr) + (static_cast<double>(v.z) <= thr) +
             (static_cast<double>(v.w) <= thr);
    }
    // blocks 0..b-1 lie entirely at or below thr; search block b
    int32_t lo = b * s, hi = min(len, (b + 1) * s);
    if (lo >= len) return len;
    while (lo < hi) {
        const int32_t mid = (lo + hi) >> 1;
        if (static_cast<double>(l[mid]) <= thr) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

struct S1Params {
    const uint8_t *rb;
    int plane1;
    int64_t nr;
    int64_t nrpad;
    float sG;
    float rmax;
    const float *c64;
    const float *psimax;
    const float *q64;
    const float *q;
    const float *reps;
    const float *radii;
    int d;
    int k;
    int64_t nq;
    int ntiles;
    float *c1_lb;
    int32_t *c1_p;
    int cap1;
    float *gamma;
    int32_t *nearest;
    int32_t *pr;
    int32_t *p3;
    int32_t *rec_cnt;
    int32_t *rec;
    int cap_rec;
    int32_t *fail;
    int32_t *tile_counter;
};

__device__ __forceinline__ int roundup16(int x) { return (x + 15) & ~15; }
__device__ __forceinline__ float max8(const float *v) {
    return fmaxf(fmaxf(fmaxf(v[0], v[1]), fmaxf(v[2], v[3])), fmaxf(fmaxf(v[4], v[5]), fmaxf(v[6], v[7])));
}
__device__ __forceinline__ float pick8(const float *v, int j) {
    const float a0 = (j & 4) ? v[4] : v[0], a1 = (j & 4) ? v[5] : v[1];
    const float a2 = (j & 4) ? v[6] : v[2], a3 = (j & 4) ? v[7] : v[3];
    const float b0 = (j & 2) ? a2 : a0, b1 = (j & 2) ? a3 : a1;
    return (j & 1) ? b1 : b0;
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
// r[j] for a runtime j in [0, 32) without local memory (select tree)
__device__ __forceinline__ uint32_t pick32u(const uint32_t (&r)[32], int j) {
    uint32_t t16[16], t8[8], t4[4];
#pragma unroll
    for (int i = 0; i < 16; ++i) t16[i] = (j & 16) ? r[i + 16] : r[i];
#pragma unroll
    for (int i = 0; i < 8; ++i) t8[i] = (j & 8) ? t16[i + 8] : t16[i];
#pragma unroll
    for (int i = 0; i < 4; ++i) t4[i] = (j & 4) ? t8[i + 4] : t8[i];
    const uint32_t a = (j & 2) ? t4[2] : t4[0], b = (j & 2) ? t4[3] : t4[1];
    return (j & 1) ? b : a;
}

// f16 hi/lo split of x: hi = f16(x), lo = f16(x - hi)
__device__ __forceinline__ void split_f16x2(float x0, float x1, uint32_t &hi, uint32_t &lo) {
    hi = sm100::pack_f16x2_sat(x0, x1);
    const __half2 h = *reinterpret_cast<const __half2 *>(&hi);
    lo = sm100::pack_f16x2_sat(x0 - __low2float(h), x1 - __high2float(h));
}

// one 128-byte row (64 f16) of hi and lo planes + aug word at column 62/63 when d <= 62
__device__ __forceinline__ void write_split_row(uint8_t *hi_row, uint8_t *lo_row, int row, const float *v, float s,
                                                bool aug_in_row, uint32_t aug) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        uint32_t wh[4], wl[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) split_f16x2(v[c * 8 + 2 * e] * s, v[c * 8 + 2 * e + 1] * s, wh[e], wl[e]);
        if (aug_in_row && c == 7) {
            wh[3] = aug;
            wl[3] = 0;
        }
        const uint32_t o = (c ^ (row & 7)) << 4;
        *reinterpret_cast<uint4 *>(hi_row + o) = make_uint4(wh[0], wh[1], wh[2], wh[3]);
        *reinterpret_cast<uint4 *>(lo_row + o) = make_uint4(wl[0], wl[1], wl[2], wl[3]);
    }
}

// ---- index preparation ------------------------------------------------------------
__global__ void rep_centre_kernel(const float *__restrict__ reps, int64_t nr, int d, float *__restrict__ c64) {
    const int k = threadIdx.x;
    if (k >= 64) return;
    double s = 0.0;
    if (k < d)
        for (int64_t p = 0; p < nr; ++p) s += reps[p * d + k];
    c64[k] = k < d ? static_cast<float>(s / static_cast<double>(nr)) : 0.f;
}

__global__ void rep_extent_kernel(const float *__restrict__ reps, int64_t nr, int d, const float *__restrict__ c64,
                                  unsigned *__restrict__ rmax_bits) {
    const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (p >= nr) return;
    double h = 0.0;
    for (int k = 0; k < d; ++k) {
        const double b = __fsub_rn(reps[p * d + k], c64[k]);
        h += b * b;
    }
    atomicMax(rmax_bits, __float_as_uint(static_cast<float>(sqrt(h)) * kUp));
}

__global__ void chunk_psimax_kernel(const float *__restrict__ radii, int64_t nr, float *__restrict__ psimax) {
    const int64_t ch = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (ch * kN >= nr) return;
    float m = 0.f;
    for (int64_t p = ch * kN; p < nr && p < (ch + 1) * kN; ++p) m = fmaxf(m, radii[p]);
    psimax[ch] = m * kUp;
}

__global__ void rep_scale_kernel(const unsigned *__restrict__ rmax_bits, float *__restrict__ stat) {
    const float r = __uint_as_float(*rmax_bits);
    int e = 0;
    if (r > 0.f) frexpf(r, &e);
    stat[0] = r > 0.f ? ldexpf(1.0f, -e) : 1.0f;
    stat[1] = r;
}

// B operand rows: f16 hi/lo of (r - c) * sG, aug = (|r - c|^2 / 2) sG^2 hi/lo
__global__ void rep_rows_kernel(const float *__restrict__ reps, int64_t nr, int d, const float *__restrict__ c64,
                                const float *__restrict__ stat, int plane1, uint8_t *__restrict__ rb) {
    const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (p >= nr) return;
    const float s = stat[0];
    float v[64];
    double h = 0.0;
#pragma unroll
    for (int k = 0; k < 64; ++k) {
        v[k] = k < d ? __fsub_rn(reps[p * d + k], c64[k]) : 0.f;
        h += static_cast<double>(v[k]) * v[k];
    }
    const float gp = static_cast<float>(h) * 0.5f * s * s;
    const __half ghi = __float2half_rn(gp);
    const __half glo = __float2half_rn(gp - __half2float(ghi));
    const uint32_t aug =
        static_cast<uint32_t>(__half_as_ushort(ghi)) | (static_cast<uint32_t>(__half_as_ushort(glo)) << 16);
    uint8_t *row = rb + p * (2 * kP0 + kP1);
    // rows are grouped in kN-row chunks: chunk base | hi plane (kN x 128) | lo plane | aug plane
    const int64_t ch = p / kN, r = p % kN;
    uint8_t *base = rb + ch * static_cast<int64_t>(kStageBytes);
    (void)row;
    write_split_row(base + r * kP0, base + kN * kP0 + r * kP0, static_cast<int>(r), v, s, !plane1, aug);
    if (plane1) {
        uint8_t *d1p = base + 2 * kN * kP0 + r * kP1;
        const int sw = static_cast<int>((r >> 2) & 1);
        *reinterpret_cast<uint4 *>(d1p + ((0 ^ sw) << 4)) = make_uint4(aug, 0, 0, 0);
        *reinterpret_cast<uint4 *>(d1p + ((1 ^ sw) << 4)) = make_uint4(0, 0, 0, 0);
    }
}

// ---- the fused stage-1 kernel ---------------------------------------------------------
template <int KT>
__global__ void __launch_bounds__(kThreads, 1) stage1_tc_kernel(const S1Params P) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024 - (sm100::smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t *sB = smem;
    uint8_t *sA = sB + kStages * kStageBytes;
    float *s_radii = reinterpret_cast<float *>(sA + 2 * kABytes);  // [nr]
    float *s_red = s_radii + kMaxRepsSmem;                          // [4] tile max of |q - c|
    uint64_t *bars = reinterpret_cast<uint64_t *>(s_red + 4);
    uint64_t *full = bars, *empty = bars + kStages, *tfull = bars + 2 * kStages, *tempty = tfull + 2;
    uint64_t *afull = tempty + 2, *aempty = afull + 2, *tile_full = aempty + 2, *tile_empty = tile_full + 2;
    uint32_t *s_tmem = reinterpret_cast<uint32_t *>(tile_empty + 2);
    int *s_tiles = reinterpret_cast<int *>(s_tmem + 1);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int64_t p = tid; p < P.nr; p += blockDim.x) s_radii[p] = P.radii[p];
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            sm100::mbar_init(&full[s], 1);
            sm100::mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            sm100::mbar_init(&tfull[b], 1);
            sm100::mbar_init(&tempty[b], 4);
            sm100::mbar_init(&afull[b], 4);
            sm100::mbar_init(&aempty[b], 1);
            sm100::mbar_init(&tile_full[b], 1);
            sm100::mbar_init(&tile_empty[b], 5);
        }
        sm100::fence_barrier_init();
    }
    if (warp == 1) sm100::tmem_alloc<256>(s_tmem);
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    const uint32_t tmem = *s_tmem;
    const int nchunks = static_cast<int>((P.nr + kN - 1) / kN);

    if (warp == 0) {
        // ===== scheduler + producer: both passes stream all representatives =====
        if (lane == 0) {
            uint32_t bi = 0;
            for (uint32_t it = 0;; ++it) {
                const uint32_t slot = it & 1;
                sm100::mbar_wait(&tile_empty[slot], ((it >> 1) & 1) ^ 1);
                const int t = atomicAdd(P.tile_counter, 1);
                const int tile = t < P.ntiles ? t : -1;
                s_tiles[slot] = tile;
                sm100::mbar_arrive(&tile_full[slot]);
                if (tile < 0) break;
                const uint32_t bytes = P.plane1 ? kStageBytes : 2 * kN * kP0;
                for (int pass = 0; pass < 2; ++pass)
                    for (int ch = 0; ch < nchunks; ++ch) {
                        const uint32_t s = bi % kStages;
                        sm100::mbar_wait(&empty[s], ((bi / kStages) & 1) ^ 1);
                        sm100::mbar_arrive_expect_tx(&full[s], bytes);
                        sm100::bulk_g2s(sB + s * kStageBytes, P.rb + static_cast<int64_t>(ch) * kStageBytes, bytes,
                                        &full[s]);
                        ++bi;
                    }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer: hi.hi + hi.lo + lo.hi (+ aug plane) =====
        if (lane == 0) {
            uint32_t bi = 0, ti = 0, ai = 0;
            for (uint32_t it = 0;; ++it) {
                const uint32_t slot = it & 1;
                sm100::mbar_wait(&tile_full[slot], (it >> 1) & 1);
                const int tile = s_tiles[slot];
                sm100::mbar_arrive(&tile_empty[slot]);
                if (tile < 0) break;
                const uint32_t a = ai & 1;
                sm100::mbar_wait(&afull[a], (ai >> 1) & 1);
                sm100::tc_fence_after();
                const uint32_t ah = sm100::smem_u32(sA + a * kABytes), al = ah + kRows * kP0;
                for (int pass = 0; pass < 2; ++pass)
                    for (int ch = 0; ch < nchunks; ++ch) {
                        const int n = min(kN, roundup16(static_cast<int>(P.nr) - ch * kN));
                        const uint32_t s = bi % kStages, tb = ti & 1;
                        sm100::mbar_wait(&full[s], (bi / kStages) & 1);
                        sm100::mbar_wait(&tempty[tb], ((ti >> 1) & 1) ^ 1);
                        sm100::tc_fence_after();
                        const uint32_t idesc = sm100::idesc_f16_f32(kRows, static_cast<uint32_t>(n));
                        const uint32_t bh = sm100::smem_u32(sB + s * kStageBytes), bl = bh + kN * kP0;
                        const uint32_t d_tmem = tmem + tb * kN;
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            sm100::umma_f16(d_tmem, sm100::umma_desc_sw128(ah + kk * 32), sm100::umma_desc_sw128(bh + kk * 32),
                                            idesc, kk > 0);
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            sm100::umma_f16(d_tmem, sm100::umma_desc_sw128(ah + kk * 32), sm100::umma_desc_sw128(bl + kk * 32),
                                            idesc, 1);
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            sm100::umma_f16(d_tmem, sm100::umma_desc_sw128(al + kk * 32), sm100::umma_desc_sw128(bh + kk * 32),
                                            idesc, 1);
                        if (P.plane1)
                            sm100::umma_f16(d_tmem, sm100::umma_desc_sw32(al + kRows * kP0),
                                            sm100::umma_desc_sw32(bl + kN * kP0), idesc, 1);
                        sm100::umma_commit(&empty[s]);
                        sm100::umma_commit(&tfull[tb]);
                        ++bi;
                        ++ti;
                    }
                sm100::umma_commit(&aempty[a]);
                ++ai;
            }
        }
    } else {
        // ===== epilogue: one query row per thread =====
        const int quad = warp & 3;
        const int row = quad * 32 + lane;
        const uint32_t lane_base = static_cast<uint32_t>(quad * 32) << 16;
        uint32_t ti = 0, ai = 0;
        for (uint32_t it = 0;; ++it) {
            const uint32_t slot = it & 1;
            sm100::mbar_wait(&tile_full[slot], (it >> 1) & 1);
            const int tile = s_tiles[slot];
            __syncwarp();
            if (lane == 0) sm100::mbar_arrive(&tile_empty[slot]);
            if (tile < 0) break;
            const int64_t qi = static_cast<int64_t>(tile) * kRows + row;
            const bool live = qi < P.nq;
            // (q - c), |q - c|^2 in fp64, tile scale sA
            float qv[64];
            double qn64 = 0.0;
            {
                const float4 *src = reinterpret_cast<const float4 *>(P.q64 + (live ? qi : 0) * 64);
                const float4 *cc = reinterpret_cast<const float4 *>(P.c64);
#pragma unroll
                for (int c = 0; c < 16; ++c) {
                    const float4 m = __ldg(cc + c);
                    const float4 t = live ? __ldg(src + c) : m;
                    qv[4 * c] = __fsub_rn(t.x, m.x);
                    qv[4 * c + 1] = __fsub_rn(t.y, m.y);
                    qv[4 * c + 2] = __fsub_rn(t.z, m.z);
                    qv[4 * c + 3] = __fsub_rn(t.w, m.w);
                }
#pragma unroll
                for (int c = 0; c < 64; ++c) qn64 += static_cast<double>(qv[c]) * qv[c];
            }
            const float qn = static_cast<float>(qn64);
            const float nqv = sqrtf(qn) * kUp;
            float tmax = nqv;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
            if (lane == 0) s_red[quad] = tmax;
            named_sync(1, 128);
            tmax = fmaxf(fmaxf(s_red[0], s_red[1]), fmaxf(s_red[2], s_red[3]));
            named_sync(1, 128);
            int e2 = 0;
            if (tmax > 0.f) frexpf(tmax, &e2);
            const float sa = tmax > 0.f ? ldexpf(1.0f, -e2) : 1.0f;
            const float scale = sa * P.sG, inv2s = 2.0f / scale;
            const float cf = sa / P.sG;
            const float acoef = (cf >= 6.103515625e-05f && cf <= 32768.0f) ? -cf : 0.0f;
            bool fail = acoef == 0.0f;
            // A operand: hi | lo | aug planes
            {
                const uint32_t a = ai & 1;
                sm100::mbar_wait(&aempty[a], ((ai >> 1) & 1) ^ 1);
                const __half ac = __float2half_rn(acoef);
                const uint32_t aug = static_cast<uint32_t>(__half_as_ushort(ac)) * 0x00010001u;
                uint8_t *abuf = sA + a * kABytes;
                write_split_row(abuf + row * kP0, abuf + kRows * kP0 + row * kP0, row, qv, sa, !P.plane1, aug);
                if (P.plane1) {
                    // the aug pairs with the B aug plane through the lo-plane descriptor slot
                    uint8_t *d1p = abuf + 2 * kRows * kP0 + row * kP1;
                    const int sw = (row >> 2) & 1;
                    *reinterpret_cast<uint4 *>(d1p + ((0 ^ sw) << 4)) = make_uint4(aug, 0, 0, 0);
                    *reinterpret_cast<uint4 *>(d1p + ((1 ^ sw) << 4)) = make_uint4(0, 0, 0, 0);
                }
                sm100::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) sm100::mbar_arrive(&afull[a]);
                ++ai;
            }
            const float rb = P.rmax;
            const float E = kC1 * nqv * rb + kC2 * (qn + rb * rb) + kC4 * rb * (2.0f / sa) + 1e-30f;

            // ---------- pass 1: bound and collect the k nearest representatives ----------
            float ubk[KT];
#pragma unroll
            for (int j = 0; j < KT; ++j) ubk[j] = __int_as_float(0x7f800000);
            float U = __int_as_float(0x7f800000);
            int count = 0;
            float *clb = P.c1_lb + (live ? qi : 0) * P.cap1;
            int32_t *cp = P.c1_p + (live ? qi : 0) * P.cap1;
            auto threshold = [&]() {
                // V >= T  <=>  lb = qn - E - 2 V / scale <= U * kTie
                const float t = 0.5f * scale * (qn - E - U * kTie);
                return t - fabsf(t) * (1.0f / 262144.0f) - 1e-30f;
            };
            float T = live ? -__int_as_float(0x7f800000) : __int_as_float(0x7f800000);
            float vbest = -__int_as_float(0x7f800000);
            auto slow8 = [&](const float *v, int col0) {
                unsigned mask = 0;
#pragma unroll
                for (int j = 0; j < 8; ++j) mask |= (v[j] >= T ? 1u : 0u) << j;
                if (col0 + 8 > P.nr) mask &= P.nr > col0 ? (0xFFu >> (8 - (P.nr - col0))) : 0u;
                while (mask) {
                    const int j = __ffs(mask) - 1;
                    mask &= mask - 1;
                    const float lb = qn - E - pick8(v, j) * inv2s;
                    if (!(lb <= U * kTie)) continue;
                    const float ub = lb + 2.0f * E;
                    if (count == P.cap1) {
                        int c2 = 0;
                        for (int e = 0; e < count; ++e)
                            if (clb[e] <= U * kTie) {
                                clb[c2] = clb[e];
                                cp[c2] = cp[e];
                                ++c2;
                            }
                        count = c2;
                        if (count == P.cap1) {
                            fail = true;
                            continue;
                        }
                    }
                    clb[count] = lb;
                    cp[count] = col0 + j;
                    ++count;
                    float x = ub;
#pragma unroll
                    for (int t = 0; t < KT; ++t) {
                        const float lo = fminf(ubk[t], x), hi = fmaxf(ubk[t], x);
                        ubk[t] = lo;
                        x = hi;
                    }
                    float kth = ubk[0];
#pragma unroll
                    for (int t = 0; t < KT; ++t)
                        if (t == P.k - 1) kth = ubk[t];
                    U = fminf(U, kth);
                    T = threshold();
                }
            };
            for (int ch = 0; ch < nchunks; ++ch) {
                const int off = ch * kN;
                const int lim = min(kN, static_cast<int>(P.nr) - off);
                const uint32_t tb = ti & 1;
                sm100::mbar_wait(&tfull[tb], (ti >> 1) & 1);
                sm100::tc_fence_after();
                for (int c0 = 0; c0 < lim; c0 += 64) {
                    uint32_t ra[32], rbv[32];
                    sm100::tmem_ld32_async(tmem + tb * kN + lane_base + c0, ra);
                    sm100::tmem_ld32_async(tmem + tb * kN + lane_base + c0 + 32, rbv);
                    sm100::tmem_wait_ld(ra);
                    sm100::tmem_tie(rbv);
                    float v[64];
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        v[j] = __uint_as_float(ra[j]);
                        v[32 + j] = __uint_as_float(rbv[j]);
                    }
                    float m8[8];
#pragma unroll
                    for (int s = 0; s < 8; ++s) m8[s] = max8(v + 8 * s);
                    if (KT == 1 && live) {
                        float mv = -__int_as_float(0x7f800000);
#pragma unroll
                        for (int s = 0; s < 8; ++s)
                            if (c0 + 8 * s + 8 <= lim) mv = fmaxf(mv, m8[s]);
                        if (mv > vbest) {
                            vbest = mv;
                            const float ub = qn + E - mv * inv2s;
                            if (ub < U) {
                                U = ub;
                                T = threshold();
                            }
                        }
                    }
#pragma unroll
                    for (int s = 0; s < 8; ++s)
                        if (m8[s] >= T) slow8(v + 8 * s, off + c0 + 8 * s);
                }
                sm100::tc_fence_before();
                __syncwarp();
                if (lane == 0) sm100::mbar_arrive(&tempty[tb]);
                ++ti;
            }
            // exact gamma_k and nearest representative from the collected candidates
            uint64_t best[KT];
#pragma unroll
            for (int j = 0; j < KT; ++j) best[j] = kEmptyKey;
            if (live && !fail) {
                const float ufin = U * kTie;
                const float *qrow = P.q + qi * P.d;
                for (int e = 0; e < count; ++e) {
                    if (!(clb[e] <= ufin)) continue;
                    const int32_t p = cp[e];
                    const float dist = exact_dist<RBC_L2>(qrow, P.reps + static_cast<int64_t>(p) * P.d, P.d);
                    const uint64_t key = pack_key(dist, static_cast<uint32_t>(p));
                    if (key < best[KT - 1]) sorted_insert<KT>(best, key);
                }
            }
            uint64_t kth_key = best[0];
#pragma unroll
            for (int t = 0; t < KT; ++t)
                if (t == P.k - 1) kth_key = best[t];
            if (live && kth_key == kEmptyKey) fail = true;
            const float g = live ? key_dist(kth_key) : 0.f;
            const float g2 = g * g;
            const float t3 = 9.0f * g2;

            // ---------- pass 2: classify every representative ----------
            int pr = 0, p3 = 0, rc = 0;
            int32_t *rec = P.rec + (live ? qi : 0) * P.cap_rec;
            for (int ch = 0; ch < nchunks; ++ch) {
                const int off = ch * kN;
                const int lim = min(kN, static_cast<int>(P.nr) - off);
                const uint32_t tb = ti & 1;
                // reps farther than max(3 gamma, gamma + max psi of the chunk) are pruned by both tests
                const float tpm = g + P.psimax[ch];
                const float thr_far = fmaxf(t3, tpm * tpm) * (1.0f + kEps) + E;  // on dt = d^2 estimate
                sm100::mbar_wait(&tfull[tb], (ti >> 1) & 1);
                sm100::tc_fence_after();
                for (int c0 = 0; c0 < lim; c0 += 32) {
                    uint32_t ra[32];
                    sm100::tmem_ld32_async(tmem + tb * kN + lane_base + c0, ra);
                    sm100::tmem_wait_ld(ra);
                    if (!live) continue;
                    const int nvalid = min(32, lim - c0);
                    const unsigned valid = nvalid == 32 ? 0xFFFFFFFFu : ((1u << nvalid) - 1u);
                    unsigned nearm = 0;
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        nearm |= ((qn - __uint_as_float(ra[j]) * inv2s) > thr_far ? 0u : 1u) << j;
                    nearm &= valid;
                    const int nfar = nvalid - __popc(nearm);
                    pr += nfar;
                    p3 += nfar;
                    while (nearm) {
                        const int j = __ffs(nearm) - 1;
                        nearm &= nearm - 1;
                        const int p = off + c0 + j;
                        const float dt = qn - __uint_as_float(pick32u(ra, j)) * inv2s;
                        const float lb = dt - E, ub = dt + E;
                        if (lb > t3 * (1.0f + kEps)) {
                            // certainly d > 3 gamma (and d > gamma); radius test decides pr
                            const float tp = g + s_radii[p];
                            const float tp2 = tp * tp;
                            if (lb > tp2 * (1.0f + kEps)) {
                                ++p3;
                                ++pr;
                            } else if (ub < tp2 * (1.0f - kEps)) {
                                ++p3;
                            } else {
                                if (rc < P.cap_rec) rec[rc] = p;  // undecided radius test
                                ++rc;
                            }
                        } else {
                            if (rc < P.cap_rec) rec[rc] = p;  // possible survivor / straddle
                            ++rc;
                        }
                    }
                }
                sm100::tc_fence_before();
                __syncwarp();
                if (lane == 0) sm100::mbar_arrive(&tempty[tb]);
                ++ti;
            }
            if (rc > P.cap_rec) fail = true;
            if (live) {
                // a failed row gets inert, in-range outputs: the batch is re-run on the
                // exact path, but stage 2 is already queued behind this kernel
                P.gamma[qi] = fail ? 0.0f : g;
                P.nearest[qi] = fail ? 0 : static_cast<int32_t>(key_id(best[0]));
                P.pr[qi] = pr;
                P.p3[qi] = p3;
                P.rec_cnt[qi] = fail ? 0 : rc;
                if (fail) atomicExch(P.fail, 1);
            }
        }
    }
    sm100::tc_fence_before();
    __syncthreads();
    if (warp == 1) sm100::tmem_dealloc<256>(tmem);
}

// Fix-up, one warp per query: exact decisions for the recorded reps, the
// 4 gamma cutoffs, the surviving segments (ascending rep position) and stats.
__global__ void __launch_bounds__(256) stage1_fixup_kernel(
    const float *__restrict__ q, const float *__restrict__ reps, int d, int64_t nq, const float *__restrict__ radii,
    const int64_t *__restrict__ offsets, const float *__restrict__ list_dists, const float *__restrict__ lskip,
    const float *__restrict__ gamma,
    const int32_t *__restrict__ nearest, const int32_t *__restrict__ rec_cnt, const int32_t *__restrict__ rec,
    int cap_rec, const int32_t *__restrict__ pr_in, const int32_t *__restrict__ p3_in, int32_t *__restrict__ nseg,
    int64_t *__restrict__ cand, int64_t *__restrict__ seg_off, int64_t *__restrict__ seg_start,
    int32_t *__restrict__ seg_len, int32_t *__restrict__ seg_list, float *__restrict__ seg_d1,
    uint64_t *__restrict__ order_key, int32_t *__restrict__ pr_out, int32_t *__restrict__ p3_out) {
    const int lane = threadIdx.x & 31;
    const int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    if (i >= nq) return;
    const double g = gamma[i], cut = 4.0 * g;
    const int n = rec_cnt[i];
    const int32_t *r = rec + i * cap_rec;
    const float *qrow = q + i * d;
    const int64_t base = i * cap_rec;
    int pr = 0, p3 = 0, ns = 0;
    long long cs = 0;
    unsigned first = 0xFFFFFFFFu;
    for (int e0 = 0; e0 < n; e0 += 32) {
        const int e = e0 + lane;
        int32_t len = 0, p = 0;
        float dist = 0.f;
        if (e < n) {
            p = r[e];
            dist = exact_dist<RBC_L2>(qrow, reps + static_cast<int64_t>(p) * d, d);
            pr += pruned_radius(dist, radii[p], g) ? 1 : 0;
            p3 += pruned_3gamma(dist, g) ? 1 : 0;
            if (survives(dist, radii[p], g))
                len = list_cutoff_skip(list_dists + offsets[p], static_cast<int32_t>(offsets[p + 1] - offsets[p]),
                                       lskip + static_cast<int64_t>(p) * 32, cut);
        }
        const unsigned bal = __ballot_sync(0xffffffffu, len > 0);
        if (len > 0) {
            const int64_t at = base + ns + __popc(bal & ((1u << lane) - 1u));
            seg_start[at] = offsets[p];
            seg_len[at] = len;
            seg_list[at] = p;
            seg_d1[at] = dist;
            cs += len;
            if (static_cast<unsigned>(p) < first) first = static_cast<unsigned>(p);
        }
        ns += __popc(bal);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        pr += __shfl_xor_sync(0xffffffffu, pr, o);
        p3 += __shfl_xor_sync(0xffffffffu, p3, o);
        cs += __shfl_xor_sync(0xffffffffu, cs, o);
        first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
    }
    if (lane == 0) {
        if (pr_out) pr_out[i] = pr_in[i] + pr;
        if (p3_out) p3_out[i] = p3_in[i] + p3;
        nseg[i] = ns;
        cand[i] = cs;
        seg_off[i] = base;
        order_key[i] = (static_cast<uint64_t>(first & 0xFFFFFFu) << 24) | (static_cast<uint32_t>(nearest[i]) & 0xFFFFFFu);
    }
}

constexpr size_t kSmemBytes = 1024 + kStages * kStageBytes + 2 * kABytes + (kMaxRepsSmem + 4) * sizeof(float) + 256;

}  // namespace

int tc1_index_prepare(rbc_index *idx, cudaStream_t st) {
    if (idx->kind != 0 || idx->metric != RBC_L2 || idx->d > 64 || idx->nr > kMaxRepsSmem) return RBC_OK;
    Tc1Index *t = new Tc1Index();
    t->plane1 = idx->d > 62;
    const int64_t nchunks = (idx->nr + kN - 1) / kN;
    t->nrpad = nchunks * kN;
    unsigned *rmax_bits = nullptr;
    bool ok = cudaMalloc(&t->rb, nchunks * kStageBytes) == cudaSuccess &&
              cudaMalloc(&t->psimax, nchunks * sizeof(float)) == cudaSuccess &&
              cudaMalloc(&t->lskip, idx->nr * 32 * sizeof(float)) == cudaSuccess &&
              cudaMalloc(&t->c64, 64 * sizeof(float)) == cudaSuccess &&
              cudaMalloc(&t->stat, 2 * sizeof(float)) == cudaSuccess &&
              cudaMalloc(&rmax_bits, sizeof(unsigned)) == cudaSuccess;
    auto cleanup = [&](int rc) {
        cudaFree(t->rb);
        cudaFree(t->psimax);
        cudaFree(t->lskip);
        cudaFree(t->c64);
        cudaFree(t->stat);
        cudaFree(rmax_bits);
        delete t;
        return rc;
    };
    if (!ok) {
        cudaGetLastError();
        return cleanup(fail(RBC_ENOMEM, "tc1 index allocation"));
    }
    cudaMemsetAsync(t->rb, 0, nchunks * kStageBytes, st);
    cudaMemsetAsync(rmax_bits, 0, sizeof(unsigned), st);
    rep_centre_kernel<<<1, 64, 0, st>>>(idx->reps, idx->nr, idx->d, t->c64);
    rep_extent_kernel<<<grid_for(idx->nr, 256), 256, 0, st>>>(idx->reps, idx->nr, idx->d, t->c64, rmax_bits);
    rep_scale_kernel<<<1, 1, 0, st>>>(rmax_bits, t->stat);
    rep_rows_kernel<<<grid_for(idx->nr, 128), 128, 0, st>>>(idx->reps, idx->nr, idx->d, t->c64, t->stat,
                                                          t->plane1 ? 1 : 0, t->rb);
    chunk_psimax_kernel<<<grid_for(nchunks, 64), 64, 0, st>>>(idx->radii, idx->nr, t->psimax);
    list_skip_kernel<<<grid_for(idx->nr * 32, 256), 256, 0, st>>>(idx->offsets, idx->list_dists, idx->nr, t->lskip);
    note_launch(6);
    float stat[2] = {1.f, 0.f};
    if (cudaMemcpyAsync(stat, t->stat, sizeof(stat), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return cleanup(fail(RBC_ECUDA, "tc1 index kernels"));
    cudaFree(rmax_bits);
    rmax_bits = nullptr;
    t->sG = stat[0];
    t->rmax = stat[1];
    idx->bytes += nchunks * kStageBytes + 66 * sizeof(float);
    idx->tc1 = t;
    return RBC_OK;
}

void tc1_index_release(rbc_index *idx) {
    Tc1Index *t = static_cast<Tc1Index *>(idx->tc1);
    if (!t) return;
    cudaFree(t->rb);
    cudaFree(t->psimax);
    cudaFree(t->lskip);
    cudaFree(t->c64);
    cudaFree(t->stat);
    delete t;
    idx->tc1 = nullptr;
}

bool tc_stage1_supported(const rbc_index *idx, int k) { return idx->tc1 != nullptr && k <= 16; }

static int g_num_sms1 = 0;

// Fused stage 1 + pruning.  Returns RBC_OK with *fallback = true when some
// row exhausted a buffer (the caller then runs the exact path).
int tc_stage1(const rbc_index *idx, const float *q, int64_t nq, int k, PruneOut &out, int32_t *fail_dev,
              cudaStream_t st) {
    const Tc1Index *t = static_cast<const Tc1Index *>(idx->tc1);
    const int ntiles = static_cast<int>((nq + kRows - 1) / kRows);
    const int cap1 = 32 + 16 * k;
    const int cap_rec = static_cast<int>(idx->nr < 512 ? idx->nr : 512);
    DevBuf<float> q64buf, c1_lb;
    DevBuf<int32_t> c1_p, nearest, pr0, p30, rec_cnt, rec, flags;
    const float *q64 = q;
    if (idx->d != 64 || (reinterpret_cast<uintptr_t>(q) & 15) != 0) {
        RBC_CHECK(q64buf.alloc(nq * 64, st));
        pad_rows64(q, nq, idx->d, q64buf.get(), st);
        q64 = q64buf.get();
    }
    RBC_CHECK(c1_lb.alloc(nq * cap1, st));
    RBC_CHECK(c1_p.alloc(nq * cap1, st));
    RBC_CHECK(nearest.alloc(nq, st));
    RBC_CHECK(pr0.alloc(nq, st));
    RBC_CHECK(p30.alloc(nq, st));
    RBC_CHECK(rec_cnt.alloc(nq, st));
    RBC_CHECK(rec.alloc(nq * cap_rec, st));
    RBC_CHECK(flags.alloc(2, st));
    RBC_CHECK(out.gamma.alloc(nq, st));
    RBC_CHECK(out.nseg.alloc(nq, st));
    RBC_CHECK(out.cand.alloc(nq, st));
    RBC_CHECK(out.seg_off.alloc(nq + 1, st));
    RBC_CHECK(out.order_key.alloc(nq, st));
    RBC_CHECK(out.seg_start.alloc(nq * cap_rec, st));
    RBC_CHECK(out.seg_len.alloc(nq * cap_rec, st));
    RBC_CHECK(out.seg_list.alloc(nq * cap_rec, st));
    RBC_CHECK(out.seg_d1.alloc(nq * cap_rec, st));
    RBC_CUDA(cudaMemsetAsync(flags.get(), 0, 2 * sizeof(int32_t), st));
    S1Params P;
    P.rb = t->rb;
    P.plane1 = t->plane1 ? 1 : 0;
    P.nr = idx->nr;
    P.nrpad = t->nrpad;
    P.sG = t->sG;
    P.rmax = t->rmax;
    P.c64 = t->c64;
    P.psimax = t->psimax;
    P.q64 = q64;
    P.q = q;
    P.reps = idx->reps;
    P.radii = idx->radii;
    P.d = idx->d;
    P.k = k;
    P.nq = nq;
    P.ntiles = ntiles;
    P.c1_lb = c1_lb.get();
    P.c1_p = c1_p.get();
    P.cap1 = cap1;
    P.gamma = out.gamma.get();
    P.nearest = nearest.get();
    P.pr = pr0.get();
    P.p3 = p30.get();
    P.rec_cnt = rec_cnt.get();
    P.rec = rec.get();
    P.cap_rec = cap_rec;
    P.fail = fail_dev;
    P.tile_counter = flags.get() + 1;
    if (g_num_sms1 == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms1, cudaDevAttrMultiProcessorCount, dev);
    }
    const unsigned grid = static_cast<unsigned>(ntiles < g_num_sms1 ? ntiles : g_num_sms1);
    auto launch = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemBytes));
        kern<<<grid, kThreads, kSmemBytes, st>>>(P);
    };
    if (k == 1) launch(stage1_tc_kernel<1>);
    else if (k <= 4) launch(stage1_tc_kernel<4>);
    else if (k <= 8) launch(stage1_tc_kernel<8>);
    else launch(stage1_tc_kernel<16>);
    RBC_LAUNCHED();
    stage1_fixup_kernel<<<grid_for(nq * 32, 256), 256, 0, st>>>(
        q, idx->reps, idx->d, nq, idx->radii, idx->offsets, idx->list_dists, t->lskip, out.gamma.get(), nearest.get(),
        rec_cnt.get(), rec.get(), cap_rec, pr0.get(), p30.get(), out.nseg.get(), out.cand.get(), out.seg_off.get(),
        out.seg_start.get(), out.seg_len.get(), out.seg_list.get(), out.seg_d1.get(), out.order_key.get(), out.pr,
        out.p3);
    RBC_LAUNCHED();
    return RBC_OK;
}

}  // namespace rbc
