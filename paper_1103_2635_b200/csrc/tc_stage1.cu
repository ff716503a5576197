// tc_stage1.cu -- exact-search stage 1 (query x representative distances),
// gamma_k and the triangle-inequality pruning, fused on the tensor cores.
//
// The reference computes every dist(q, r) exactly (search.py:178), takes the
// k-th smallest as gamma_k (:181), and keeps r iff
//   d <= 3 gamma  and  (d < gamma + psi_r  or  d <= gamma)      (:62-74)
// counting the two pruning tests (:194-195).  Here each 128-query tile is
// multiplied against all representatives with one tcgen05.mma kind::f16 per
// K=16 slice: operands centred on the representatives' mean c, the per-rep
// term |r - c|^2 / 2 folded into the MMA as two extra K columns (as in
// tc_stage2.cu), so every d^2 is known inside a rigorous interval
// [dt - E, dt + E].  The accumulator row of |R| columns does not fit TMEM, so
// the representatives stream through in 128-column chunks:
//   k > 1, pass 1: the k smallest upper bounds give U_k >= gamma_k^2; every
//           rep with lb <= U_k is buffered as a gamma candidate, and
//           gamma_k^2 lies in [U_k - 2E, U_k];
//   k > 1, pass 2: every rep is classified against 3 gamma and gamma + psi
//           with that gamma interval.  Far reps (almost all) are only
//           counted, 8 at a time through a max-reduce; the rest is recorded
//           with its estimate.
//   k = 1: one pass.  The running bound starts at the query's distance to its
//           pilot (pilot_key_kernel, an upper bound of gamma^2) and tightens
//           block by block; each block is classified against the far test
//           with the current bound right after (the bound only decreases, so
//           "far" stays certain under the final gamma).
// No fp64 work happens here.  The fix-up kernel (an 8-lane group per query)
// turns the gamma candidates into the exact gamma_k and nearest rep with the
// reference arithmetic, decides the recorded reps exactly, computes the
// 4 gamma cutoffs and emits the surviving segments.  No |Q| x |R| distance
// matrix is materialised.  Any row that exhausts a buffer raises a flag and
// the caller recomputes the batch with the exact path (search.cu), so the
// result is always the reference's.
#include <cub/cub.cuh>

#include <cstdio>
#include <cstdlib>
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
constexpr int kN = 128;        // representatives per chunk (UMMA N)
constexpr int kStages = 3;
constexpr int kThreads = 192;  // producer, MMA, 4 epilogue warps
constexpr int kP0 = 128, kP1 = 32;
// per chunk: plane 0 (kN rows x 128 B, SW128: 64 f16, aug in columns 62/63 when
// d <= 62) | plane 1 (kN rows x 32 B, SW32: the aug pair, d > 62 only)
constexpr int kStageBytes = kN * (kP0 + kP1);
constexpr int kABytes = kRows * (kP0 + kP1);
constexpr int kMaxRepsSmem = 6144;  // radii staged in shared memory

// error bound of the centred f16 expanded form (same derivation as tc_stage2.cu:
// f16 rounding of a and b, fp32 accumulation of <= 80 products, factor-2 safety)
constexpr float kC1 = 4.0f * (1.0f / 1024.0f + 128.0f / 4194304.0f);
constexpr float kC2 = 1.0f / 1048576.0f;
constexpr float kC4 = 1.0f / 262144.0f;
constexpr float kUp = 1.0f + 1.0f / 1048576.0f;
constexpr float kTie = 1.0f + 1.0f / 524288.0f;
constexpr float kEps = 1.0f / 262144.0f;  // relative slack of the interval classification
constexpr float kCq = 1.0f / 65536.0f;    // fp32 |q - c|^2 (<= 66 ulps) and its square root

struct Tc1Index {
    int64_t nrpad = 0;
    bool plane1 = false;
    uint8_t *rb = nullptr;   // [nchunks] x kStageBytes, pre-swizzled f16 rows of (r - c) sG (+ aug)
    float *c64 = nullptr;    // [64] centre (mean of the reps), zero padded
    float *stat = nullptr;   // [2] sG, rmax (max |r - c|, rounded up)
    float *psimax = nullptr; // [nchunks] largest list radius of each rep chunk
    float *lskip = nullptr;  // [nr][32] list_dists at the end of each of 32 equal blocks (cutoff skip table)
    float *reps64 = nullptr; // [nr][64] representatives, zero padded (16-byte rows for the fix-up)
    int32_t *pilots = nullptr; // [kPilots] farthest-point sample of the reps (query ordering)
    uint4 *prow = nullptr;     // [kPilots * 8] pilot rows as f16
    float *pnorm = nullptr;    // [kPilots] |pilot|^2 / 2
    float sG = 1.f, rmax = 0.f;
};

constexpr int kPilots = 64;  // query-ordering pilots (farthest-point sample of the reps)

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
    float sG;
    float rmax;
    const float *c64;
    const float *psimax;
    const float *pd2;       // [nq] k = 1: upper bound of gamma_1^2 from the query's pilot
    const float *q64;
    const int32_t *qorder;  // tile slot -> query id (queries sorted by nearest pilot)
    const float *radii;
    int k;
    int64_t nq;
    int ntiles;
    float *c1_lb;      // [nq][cap1] gamma-candidate lower bounds
    int32_t *c1_p;     // [nq][cap1] their rep positions
    int cap1;
    int32_t *c1_cnt;   // [nq] buffered gamma candidates (-1: row failed)
    float *c1_u;       // [nq] U_k * kTie: a candidate matters iff lb <= c1_u
    int32_t *pr;       // [nq] reps decided here as pruned by the radius test
    int32_t *p3;       // [nq] ... by the 3 gamma test
    int32_t *rec_cnt;  // [nq]
    int32_t *rec;      // [nq][cap_rec] recorded (not certainly far) reps
    float *rec_dt;     // [nq][cap_rec] their d^2 estimate (true d^2 within +-rec_e)
    float *rec_e;      // [nq] the row's error bound E
    int cap_rec;
    int32_t *fail;
    int32_t *tile_counter;
    unsigned long long *timing;  // diagnostic [12] summed role wait cycles (nullptr = off)
};

__device__ __forceinline__ int roundup16(int x) { return (x + 15) & ~15; }
__device__ __forceinline__ float max8(const float *v) { return sm100::max8(v); }
__device__ __forceinline__ float pick8(const float *v, int j) {
    const float a0 = (j & 4) ? v[4] : v[0], a1 = (j & 4) ? v[5] : v[1];
    const float a2 = (j & 4) ? v[6] : v[2], a3 = (j & 4) ? v[7] : v[3];
    const float b0 = (j & 2) ? a2 : a0, b1 = (j & 2) ? a3 : a1;
    return (j & 1) ? b1 : b0;
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// one 128-byte row (64 f16 of v * s), aug word at columns 62/63 when d <= 62
__device__ __forceinline__ void write_row(uint8_t *dst, int row, const float *v, float s, bool aug_in_row,
                                          uint32_t aug) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        uint32_t w[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) w[e] = sm100::pack_f16x2_sat(v[c * 8 + 2 * e] * s, v[c * 8 + 2 * e + 1] * s);
        if (aug_in_row && c == 7) w[3] = aug;
        *reinterpret_cast<uint4 *>(dst + ((c ^ (row & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

// aug pair in its own 32-byte SW32 row (d > 62)
__device__ __forceinline__ void write_aug_row(uint8_t *dst, int row, uint32_t aug) {
    const int sw = (row >> 2) & 1;
    *reinterpret_cast<uint4 *>(dst + ((0 ^ sw) << 4)) = make_uint4(aug, 0, 0, 0);
    *reinterpret_cast<uint4 *>(dst + ((1 ^ sw) << 4)) = make_uint4(0, 0, 0, 0);
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

// B operand rows: f16 of (r - c) sG, aug = (|r - c|^2 / 2) sG^2 as an f16 hi/lo pair
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
    const int64_t ch = p / kN, r = p % kN;
    uint8_t *base = rb + ch * static_cast<int64_t>(kStageBytes);
    write_row(base + r * kP0, static_cast<int>(r), v, s, !plane1, aug);
    if (plane1) write_aug_row(base + kN * kP0 + r * kP1, static_cast<int>(r), aug);
}

// Pilot reps by farthest-point sampling (one block): start at rep 0, then repeatedly the
// rep farthest from the chosen set.  With clustered data the pilots land one per region,
// so queries sorted by nearest pilot fill tiles from a single region.
__global__ void __launch_bounds__(1024) pilot_fps_kernel(const float *__restrict__ reps64, int64_t nr, int npilot,
                                                         int32_t *__restrict__ pilots) {
    extern __shared__ float mind[];  // [nr]
    __shared__ unsigned long long s_best;
    __shared__ int s_last;
    for (int64_t p = threadIdx.x; p < nr; p += blockDim.x) mind[p] = __int_as_float(0x7f800000);
    if (threadIdx.x == 0) {
        s_last = 0;
        pilots[0] = 0;
    }
    __syncthreads();
    for (int it = 1; it < npilot; ++it) {
        const float4 *l4 = reinterpret_cast<const float4 *>(reps64 + static_cast<int64_t>(s_last) * 64);
        if (threadIdx.x == 0) s_best = 0;
        __syncthreads();
        unsigned long long best = 0;
        for (int64_t p = threadIdx.x; p < nr; p += blockDim.x) {
            const float4 *r4 = reinterpret_cast<const float4 *>(reps64 + p * 64);
            float a = 0.f;
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                const float4 x = __ldg(r4 + c), y = __ldg(l4 + c);
                const float t0 = x.x - y.x, t1 = x.y - y.y, t2 = x.z - y.z, t3 = x.w - y.w;
                a = fmaf(t0, t0, fmaf(t1, t1, fmaf(t2, t2, fmaf(t3, t3, a))));
            }
            const float m = fminf(mind[p], a);
            mind[p] = m;
            // farthest first, lowest position on ties (non-negative floats order as their bits)
            const unsigned long long key = (static_cast<unsigned long long>(__float_as_uint(m)) << 32) |
                                           (0xFFFFFFFFu - static_cast<unsigned>(p));
            best = key > best ? key : best;
        }
        atomicMax(&s_best, best);
        __syncthreads();
        if (threadIdx.x == 0) {
            const int p = static_cast<int>(0xFFFFFFFFu - static_cast<unsigned>(s_best & 0xFFFFFFFFu));
            pilots[it] = p;
            s_last = p;
        }
        __syncthreads();
    }
}

// Query ordering: key = nearest of kPilots spread reps.  Approximate on purpose
// (f16 products, max of q.r - |r|^2/2): it only decides which queries share a
// tile, never a result.  Queries of one region then share their near reps, so
// the per-tile slow paths run in lockstep.
// pilot rows as f16 (64 per row) and |r|^2 / 2, once per index
__global__ void pilot_rows_kernel(const float *__restrict__ reps64, const int32_t *__restrict__ pilots, int npilot,
                                  uint4 *__restrict__ prow, float *__restrict__ pnorm) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < npilot * 8) {
        const int j = t >> 3, c = t & 7;
        const float4 *row = reinterpret_cast<const float4 *>(reps64 + static_cast<int64_t>(pilots[j]) * 64) + 2 * c;
        const float4 a = __ldg(row), b = __ldg(row + 1);
        prow[t] = make_uint4(sm100::pack_f16x2_sat(a.x, a.y), sm100::pack_f16x2_sat(a.z, a.w),
                             sm100::pack_f16x2_sat(b.x, b.y), sm100::pack_f16x2_sat(b.z, b.w));
    }
    if (t < npilot) {
        const float4 *row = reinterpret_cast<const float4 *>(reps64 + static_cast<int64_t>(pilots[t]) * 64);
        float n = 0.f;
#pragma unroll
        for (int c = 0; c < 16; ++c) {
            const float4 v = __ldg(row + c);
            n = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, n))));
        }
        pnorm[t] = 0.5f * n;
    }
}

// Query ordering key: nearest of the kPilots pilots, as a small tensor-core GEMM
// (mma.sync m16n8k16, f16 inputs, fp32 accumulate): one warp scores 16 queries against
// all 64 pilots (argmax of q.p - |p|^2 / 2).  Approximate on purpose: it only decides
// which queries share a tile, never a result.
constexpr int kPilotWarps = 8;  // 128 queries per block
__device__ __forceinline__ uint32_t f2h2(float a, float b) { return sm100::pack_f16x2_sat(a, b); }

__global__ void __launch_bounds__(kPilotWarps * 32) pilot_key_kernel(const float *__restrict__ q64, int64_t nq,
                                                                    const uint4 *__restrict__ prow,
                                                                    const float *__restrict__ pnorm, int npilot,
                                                                    const float *__restrict__ reps64,
                                                                    const int32_t *__restrict__ pilots,
                                                                    uint32_t *__restrict__ key,
                                                                    unsigned *__restrict__ hist,
                                                                    float *__restrict__ pd2) {
    // pilot rows, 64 f16 (32 words) each, at a 36-word stride: the 8 row groups of an mma
    // B fragment then read 8 different bank quads (a 32-word stride is an 8-way conflict);
    // absent pilots zero
    constexpr int kSpStride = 36;
    __shared__ __align__(16) uint32_t sp[kPilots * kSpStride];
    __shared__ float sn[kPilots];
    __shared__ unsigned sh[kPilots];
    for (int t = threadIdx.x; t < kPilots * 8; t += blockDim.x) {
        const uint4 v = t < npilot * 8 ? prow[t] : make_uint4(0, 0, 0, 0);
        reinterpret_cast<uint4 *>(sp)[(t >> 3) * (kSpStride / 4) + (t & 7)] = v;
    }
    for (int j = threadIdx.x; j < kPilots; j += blockDim.x) {
        sh[j] = 0;
        sn[j] = j < npilot ? pnorm[j] : __int_as_float(0x7f800000);  // absent pilots never win
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
    const int64_t r0 = (static_cast<int64_t>(blockIdx.x) * kPilotWarps + warp) * 16;
    const int64_t ra = r0 + g < nq ? r0 + g : nq - 1, rb = r0 + g + 8 < nq ? r0 + g + 8 : nq - 1;
    const float *qa = q64 + ra * 64, *qb = q64 + rb * 64;
    float acc[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
        const int c0 = 16 * ks + 2 * t4;
        const float2 x0 = __ldg(reinterpret_cast<const float2 *>(qa + c0));
        const float2 x1 = __ldg(reinterpret_cast<const float2 *>(qb + c0));
        const float2 x2 = __ldg(reinterpret_cast<const float2 *>(qa + c0 + 8));
        const float2 x3 = __ldg(reinterpret_cast<const float2 *>(qb + c0 + 8));
        const uint32_t a0 = f2h2(x0.x, x0.y), a1 = f2h2(x1.x, x1.y), a2 = f2h2(x2.x, x2.y), a3 = f2h2(x3.x, x3.y);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t *prow_n = sp + (8 * j + g) * kSpStride;  // pilot n = 8 j + g, words = dim pairs
            const uint32_t b0 = prow_n[(16 * ks + 2 * t4) >> 1], b1 = prow_n[(16 * ks + 8 + 2 * t4) >> 1];
            asm volatile(
                "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%0,%1,%2,%3};"
                : "+f"(acc[j][0]), "+f"(acc[j][1]), "+f"(acc[j][2]), "+f"(acc[j][3])
                : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
        }
    }
    // rows g (acc[.][0..1]) and g + 8 (acc[.][2..3]); columns 8 j + 2 t4 (+1)
    float bestA = -__int_as_float(0x7f800000), bestB = bestA;
    int jA = 0, jB = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int n = 8 * j + 2 * t4 + h;
            const float sA = acc[j][h] - sn[n], sB = acc[j][2 + h] - sn[n];
            if (sA > bestA) bestA = sA, jA = n;
            if (sB > bestB) bestB = sB, jB = n;
        }
#pragma unroll
    for (int o = 1; o < 4; o <<= 1) {  // the 4 lanes of the row group
        const float vA = __shfl_xor_sync(0xffffffffu, bestA, o), vB = __shfl_xor_sync(0xffffffffu, bestB, o);
        const int iA = __shfl_xor_sync(0xffffffffu, jA, o), iB = __shfl_xor_sync(0xffffffffu, jB, o);
        if (vA > bestA || (vA == bestA && iA < jA)) bestA = vA, jA = iA;
        if (vB > bestB || (vB == bestB && iB < jB)) bestB = vB, jB = iB;
    }
    // |q - chosen pilot|^2 in fp32 (the 4 lanes of the row group, 16 coordinates each),
    // rounded up by 2^-16 relative (the fp32 error is <= 66 * 2^-24): an upper bound of
    // gamma_1^2 that seeds stage 1's running bound
    {
        const float4 *pa = reinterpret_cast<const float4 *>(reps64 + static_cast<int64_t>(pilots[jA]) * 64) + 4 * t4;
        const float4 *pb = reinterpret_cast<const float4 *>(reps64 + static_cast<int64_t>(pilots[jB]) * 64) + 4 * t4;
        const float4 *xa = reinterpret_cast<const float4 *>(qa) + 4 * t4;
        const float4 *xb = reinterpret_cast<const float4 *>(qb) + 4 * t4;
        float sa = 0.f, sb = 0.f, mx = 0.f;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const float4 u = __ldg(xa + c), v = __ldg(pa + c), w = __ldg(xb + c), z = __ldg(pb + c);
            const float a0 = u.x - v.x, a1 = u.y - v.y, a2 = u.z - v.z, a3 = u.w - v.w;
            const float b0 = w.x - z.x, b1 = w.y - z.y, b2 = w.z - z.z, b3 = w.w - z.w;
            sa = fmaf(a0, a0, fmaf(a1, a1, fmaf(a2, a2, fmaf(a3, a3, sa))));
            sb = fmaf(b0, b0, fmaf(b1, b1, fmaf(b2, b2, fmaf(b3, b3, sb))));
            mx = fmaxf(mx, fmaxf(fmaxf(fabsf(u.x), fabsf(u.y)), fmaxf(fabsf(u.z), fabsf(u.w))));
            mx = fmaxf(mx, fmaxf(fmaxf(fabsf(w.x), fabsf(w.y)), fmaxf(fabsf(w.z), fabsf(w.w))));
            if (u.x != u.x || u.y != u.y || u.z != u.z || u.w != u.w || w.x != w.x || w.y != w.y || w.z != w.z ||
                w.w != w.w)
                mx = __int_as_float(0x7f800000);
        }
        // the tensor-core bounds' range (tc_scan.cuh kTcMaxAbs): larger queries -> exact path
        // (hist[2 kPilots]; pilot_scatter_kernel turns it into stage 1's failure flag)
        if (!(mx <= kTcMaxAbs)) atomicOr(hist + 2 * kPilots, 1u);
#pragma unroll
        for (int o = 1; o < 4; o <<= 1) {
            sa += __shfl_xor_sync(0xffffffffu, sa, o);
            sb += __shfl_xor_sync(0xffffffffu, sb, o);
        }
        if (t4 == 0) {
            if (r0 + g < nq) pd2[r0 + g] = sa * (1.0f + 1.0f / 65536.0f) + 1e-30f;
            if (r0 + g + 8 < nq) pd2[r0 + g + 8] = sb * (1.0f + 1.0f / 65536.0f) + 1e-30f;
        }
    }
    if (t4 == 0) {
        if (r0 + g < nq) {
            key[r0 + g] = static_cast<uint32_t>(jA);
            atomicAdd(&sh[jA], 1u);
        }
        if (r0 + g + 8 < nq) {
            key[r0 + g + 8] = static_cast<uint32_t>(jB);
            atomicAdd(&sh[jB], 1u);
        }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < npilot; j += blockDim.x)
        if (sh[j]) atomicAdd(&hist[j], sh[j]);
}

// Query order from the pilot keys: a counting sort over the kPilots buckets (bucket
// starts = exclusive scan of the histogram; each block claims a contiguous range per
// bucket).  Order inside a bucket follows the blocks' claims -- it only shapes tiles.
__global__ void __launch_bounds__(128) pilot_scatter_kernel(const uint32_t *__restrict__ key, int64_t nq, int npilot,
                                                            const unsigned *__restrict__ hist,
                                                            unsigned *__restrict__ cursor, int32_t *__restrict__ qorder,
                                                            int32_t *__restrict__ zero2,
                                                            unsigned long long *__restrict__ zero64,
                                                            int32_t *__restrict__ fail2) {
    __shared__ unsigned s_start[kPilots], s_cnt[kPilots], s_base[kPilots];
    // stage 1's two flags, its failure words and stage 2's work counter start at zero here
    // (no memset nodes; every writer of them runs after this kernel)
    if (blockIdx.x == 0 && threadIdx.x < 2) zero2[threadIdx.x] = 0;
    if (blockIdx.x == 0 && threadIdx.x == 2) *zero64 = 0ull;
    if (blockIdx.x == 0 && threadIdx.x >= 4 && threadIdx.x < 6)  // [0]: queries beyond the tensor-core range
        fail2[threadIdx.x - 4] = threadIdx.x == 4 && cursor[kPilots] != 0u ? 1 : 0;
    if (threadIdx.x == 0) {
        unsigned run = 0;
        for (int j = 0; j < npilot; ++j) {
            s_start[j] = run;
            run += hist[j];
        }
    }
    for (int j = threadIdx.x; j < kPilots; j += blockDim.x) s_cnt[j] = 0;
    __syncthreads();
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int b = i < nq ? static_cast<int>(key[i]) : -1;
    const unsigned r = b >= 0 ? atomicAdd(&s_cnt[b], 1u) : 0u;
    __syncthreads();
    for (int j = threadIdx.x; j < npilot; j += blockDim.x)
        if (s_cnt[j]) s_base[j] = s_start[j] + atomicAdd(&cursor[j], s_cnt[j]);
    __syncthreads();
    if (b >= 0) qorder[s_base[b] + r] = static_cast<int32_t>(i);
}

__global__ void pad_reps64_kernel(const float *__restrict__ src, int64_t rows, int d, float *__restrict__ dst) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t >= rows * 64) return;
    const int64_t r = t >> 6;
    const int c = static_cast<int>(t & 63);
    dst[t] = c < d ? src[r * d + c] : 0.f;
}

// Diagnostic role timing (build with -DRBC_S1_TIMING, run with RBC_DEBUG_S1=1)
#ifdef RBC_S1_TIMING
__device__ __forceinline__ void s1_wait_t(uint64_t *bar, uint32_t parity, unsigned long long &acc) {
    const unsigned long long t0 = clock64();
    sm100::mbar_wait(bar, parity);
    acc += clock64() - t0;
}
#define S1_WAIT(bar, parity, slot) s1_wait_t(bar, parity, tw[slot])
#else
#define S1_WAIT(bar, parity, slot) sm100::mbar_wait(bar, parity)
#endif

#ifdef RBC_S1_NOEPI
#define S1_LIM(x) 0  // diagnostic: pipeline without epilogue work (results invalid)
#else
#define S1_LIM(x) (x)
#endif

// ---- the fused stage-1 kernel ---------------------------------------------------------
template <int KT>
__global__ void __launch_bounds__(kThreads, 2) stage1_tc_kernel(const S1Params P) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024 - (sm100::smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t *sB = smem;
    uint8_t *sA = sB + kStages * kStageBytes;
    float *s_radii = reinterpret_cast<float *>(sA + 2 * kABytes);  // [nr]
    float *s_red = s_radii + ((P.nr + 3) & ~int64_t(3));            // [4] tile max of |q - c|
    uint64_t *bars = reinterpret_cast<uint64_t *>(s_red + 4);
    uint64_t *full = bars, *empty = bars + kStages, *tfull = bars + 2 * kStages, *tempty = tfull + 2;
    uint64_t *afull = tempty + 2, *aempty = afull + 2, *tile_full = aempty + 2, *tile_empty = tile_full + 2;
    uint32_t *s_tmem = reinterpret_cast<uint32_t *>(tile_empty + 2);
    int *s_tiles = reinterpret_cast<int *>(s_tmem + 1);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
#ifdef RBC_S1_TIMING
    unsigned long long tw[14] = {};
    const unsigned long long t_start = clock64();
#endif
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
        // ===== scheduler + producer: the tile's query rows (gathered through qorder, one
        // 256-byte bulk copy per row, all lanes), then both passes of the representatives =====
        uint32_t bi = 0;
        for (uint32_t it = 0;; ++it) {
            const uint32_t slot = it & 1;
            int tile = 0;
            if (lane == 0) {
                S1_WAIT(&tile_empty[slot], ((it >> 1) & 1) ^ 1, 0);
                const int t = atomicAdd(P.tile_counter, 1);
                tile = t < P.ntiles ? t : -1;
                s_tiles[slot] = tile;
                sm100::mbar_arrive(&tile_full[slot]);
            }
            tile = __shfl_sync(0xffffffffu, tile, 0);
            if (tile < 0) break;
            if (lane == 0) {
                const uint32_t bytes = P.plane1 ? kStageBytes : kN * kP0;
                for (int pass = 0; pass < (P.k == 1 ? 1 : 2); ++pass)
                    for (int ch = 0; ch < nchunks; ++ch) {
                        const uint32_t s = bi % kStages;
                        S1_WAIT(&empty[s], ((bi / kStages) & 1) ^ 1, 1);
                        sm100::mbar_arrive_expect_tx(&full[s], bytes);
                        sm100::bulk_g2s(sB + s * kStageBytes, P.rb + static_cast<int64_t>(ch) * kStageBytes, bytes,
                                        &full[s]);
                        ++bi;
                    }
            }
            __syncwarp();
        }
    } else if (warp == 1) {
        // ===== MMA issuer: 4 x K16 over plane 0 (+ the aug plane) =====
        if (lane == 0) {
            uint32_t bi = 0, ti = 0, ai = 0;
            for (uint32_t it = 0;; ++it) {
                const uint32_t slot = it & 1;
                S1_WAIT(&tile_full[slot], (it >> 1) & 1, 2);
                const int tile = s_tiles[slot];
                sm100::mbar_arrive(&tile_empty[slot]);
                if (tile < 0) break;
                const uint32_t a = ai & 1;
                S1_WAIT(&afull[a], (ai >> 1) & 1, 3);
                sm100::tc_fence_after();
                const uint32_t a0 = sm100::smem_u32(sA + a * kABytes);
                for (int pass = 0; pass < (P.k == 1 ? 1 : 2); ++pass)
                    for (int ch = 0; ch < nchunks; ++ch) {
                        const int n = min(kN, roundup16(static_cast<int>(P.nr) - ch * kN));
                        const uint32_t s = bi % kStages, tb = ti & 1;
                        S1_WAIT(&full[s], (bi / kStages) & 1, 4);
                        S1_WAIT(&tempty[tb], ((ti >> 1) & 1) ^ 1, 5);
                        sm100::tc_fence_after();
                        const uint32_t idesc = sm100::idesc_f16_f32(kRows, static_cast<uint32_t>(n));
                        const uint32_t b0 = sm100::smem_u32(sB + s * kStageBytes);
                        const uint32_t d_tmem = tmem + tb * kN;
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            sm100::umma_f16(d_tmem, sm100::umma_desc_sw128(a0 + kk * 32), sm100::umma_desc_sw128(b0 + kk * 32),
                                            idesc, kk > 0);
                        if (P.plane1)
                            sm100::umma_f16(d_tmem, sm100::umma_desc_sw32(a0 + kRows * kP0),
                                            sm100::umma_desc_sw32(b0 + kN * kP0), idesc, 1);
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
            S1_WAIT(&tile_full[slot], (it >> 1) & 1, 6);
            const int tile = s_tiles[slot];
            __syncwarp();
            if (lane == 0) sm100::mbar_arrive(&tile_empty[slot]);
            if (tile < 0) break;
            const int64_t slot_i = static_cast<int64_t>(tile) * kRows + row;
            const bool live = slot_i < P.nq;
            const int64_t qi = live ? P.qorder[slot_i] : 0;
            // (q - c) from the staged row, |q - c|^2 (fp32: relative error <= 66 * 2^-24, covered by kCq)
            float qv[64];
            float qn;
            {
                const float4 *src = reinterpret_cast<const float4 *>(P.q64 + qi * 64);
                const float4 *cc = reinterpret_cast<const float4 *>(P.c64);
                float n0 = 0.f, n1 = 0.f;
#pragma unroll
                for (int c = 0; c < 16; ++c) {
                    const float4 m = __ldg(cc + c);
                    const float4 t = live ? __ldg(src + c) : m;
                    qv[4 * c] = __fsub_rn(t.x, m.x);
                    qv[4 * c + 1] = __fsub_rn(t.y, m.y);
                    qv[4 * c + 2] = __fsub_rn(t.z, m.z);
                    qv[4 * c + 3] = __fsub_rn(t.w, m.w);
                    n0 = fmaf(qv[4 * c], qv[4 * c], fmaf(qv[4 * c + 1], qv[4 * c + 1], n0));
                    n1 = fmaf(qv[4 * c + 2], qv[4 * c + 2], fmaf(qv[4 * c + 3], qv[4 * c + 3], n1));
                }
                qn = n0 + n1;
            }
            const float nqv = sqrtf(qn) * (1.0f + kCq);
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
            // A operand: f16 rows of (q - c) sA, aug = -sA / sG in the aug columns
            {
                const uint32_t a = ai & 1;
                S1_WAIT(&aempty[a], ((ai >> 1) & 1) ^ 1, 7);
                const __half ac = __float2half_rn(acoef);
                const uint32_t aug = static_cast<uint32_t>(__half_as_ushort(ac)) * 0x00010001u;
                uint8_t *abuf = sA + a * kABytes;
                write_row(abuf + row * kP0, row, qv, sa, !P.plane1, aug);
                if (P.plane1) write_aug_row(abuf + kRows * kP0 + row * kP1, row, aug);
                sm100::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) sm100::mbar_arrive(&afull[a]);
                ++ai;
            }
            const float rb = P.rmax;
            const float E = kC1 * nqv * rb + kC2 * (qn + rb * rb) + kCq * qn + kC4 * rb * (2.0f / sa) + 1e-30f;

            // ---------- pass 1: bound and collect the gamma candidates ----------
            // Every rep with lb <= U (U = running k-th smallest upper bound) is buffered;
            // the bound is tightened from group maxima (each group's best is a distinct rep).
            float ubk[KT];
#pragma unroll
            for (int j = 0; j < KT; ++j) ubk[j] = __int_as_float(0x7f800000);
            float U = __int_as_float(0x7f800000);
            int count = 0;
            float *clb = P.c1_lb + (live ? qi : 0) * P.cap1;
            int32_t *cp = P.c1_p + (live ? qi : 0) * P.cap1;
            auto threshold = [&]() {
                // V >= T  <=>  lb = qn - E - 2 V / scale <= U * kTie   (loosened by 2^-18 relative)
                const float t = 0.5f * scale * (qn - E - U * kTie);
                return t - fabsf(t) * (1.0f / 262144.0f) - 1e-30f;
            };
            const float lb0 = qn - E;  // lb(V) = lb0 - V * inv2s
            float T = live ? -__int_as_float(0x7f800000) : __int_as_float(0x7f800000);
            // k = 1: one pass.  The running bound starts at the pilot's distance (an upper bound
            // of gamma_1^2), so each block can be classified against the far test right away --
            // with a bound that only decreases, "far" stays certain under the final gamma, and
            // the recorded rest is re-classified by the fix-up.  k > 1: two passes.
            constexpr bool kSingle = KT == 1;
            if (kSingle && live) {
                U = P.pd2[qi];
                T = threshold();
            }
            int pr = 0, p3 = 0, rc = 0;
            int32_t *rec = P.rec + (live ? qi : 0) * P.cap_rec;
            float *rdt = P.rec_dt + (live ? qi : 0) * P.cap_rec;
            for (int ch = 0; ch < nchunks; ++ch) {
                const int off = ch * kN;
                const int lim = min(kN, static_cast<int>(P.nr) - off);
                const uint32_t tb = ti & 1;
                const float psic = P.psimax[ch];
                S1_WAIT(&tfull[tb], (ti >> 1) & 1, 8);
                sm100::tc_fence_after();
                for (int c0 = 0; c0 < S1_LIM(lim); c0 += 64) {
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
                    // bound from the valid groups' maxima first (k = 1: the block's best)
                    if (KT == 1) {
                        float mv = -__int_as_float(0x7f800000);
#pragma unroll
                        for (int s = 0; s < 8; ++s)
                            if (c0 + 8 * s + 8 <= lim) mv = fmaxf(mv, m8[s]);
                        const float ub = fmaf(-mv, inv2s, lb0) + 2.0f * E;
                        if (live && ub < U) {
                            U = ub;
                            T = threshold();
                        }
                    }
                    unsigned gm = 0;  // groups that may hold a candidate
#pragma unroll
                    for (int s = 0; s < 8; ++s) gm |= (m8[s] >= T ? 1u : 0u) << s;
                    // rare path, compact code: walk the groups flagged by any lane (warp-uniform),
                    // re-reading each group's 8 columns from TMEM
                    unsigned gu = __reduce_or_sync(0xffffffffu, gm);
                    while (gu) {
                        const int s = __ffs(gu) - 1;
                        gu &= gu - 1;
                        float x[8];
                        sm100::tmem_ld8(tmem + tb * kN + lane_base + c0 + 8 * s, x);
                        bool take = (gm & (1u << s)) != 0;
                        const int g0 = off + c0 + 8 * s;
                        if (take && count + 8 > P.cap1) {  // compact: drop entries that can no longer qualify
                            int c2 = 0;
                            for (int e = 0; e < count; ++e)
                                if (clb[e] <= U * kTie) {
                                    clb[c2] = clb[e];
                                    cp[c2] = cp[e];
                                    ++c2;
                                }
                            count = c2;
                            if (count + 8 > P.cap1) {
                                fail = true;
                                take = false;
#ifdef RBC_FAIL_WHY
                                atomicOr(P.fail + 1, 1);
#endif
                            }
                        }
                        unsigned hit = 0;  // the group's elements that qualify, then only those
#pragma unroll
                        for (int j = 0; j < 8; ++j) hit |= (take && x[j] >= T && g0 + j < P.nr ? 1u : 0u) << j;
                        while (hit) {
                            const int j = __ffs(hit) - 1;
                            hit &= hit - 1;
                            {
                                const float lb = fmaf(-pick8(x, j), inv2s, lb0);
                                clb[count] = lb;
                                cp[count] = g0 + j;
                                ++count;
                                if (KT > 1) {
                                    float y = lb + 2.0f * E;
#pragma unroll
                                    for (int t = 0; t < KT; ++t) {
                                        const float lo = fminf(ubk[t], y), hi = fmaxf(ubk[t], y);
                                        ubk[t] = lo;
                                        y = hi;
                                    }
                                }
                            }
                        }
                        if (KT > 1 && take) {
                            float kth = ubk[KT - 1];  // KT = 10 serves k = 10 only
                            if (KT != 10) {
#pragma unroll
                                for (int t = 0; t < KT; ++t)
                                    if (t == P.k - 1) kth = ubk[t];
                            }
                            U = fminf(U, kth);
                            T = threshold();
                        }
                        __syncwarp();
                    }
                    if (kSingle) {  // the same block against the far test with the current bound
                        const float ghi = sqrtf(U * kTie) * kUp;
                        const float tpm = ghi + psic;
                        const float thr_far = fmaxf(9.0f * ghi * ghi * (1.0f + kEps), tpm * tpm * (1.0f + kEps));
                        const float tf = 0.5f * scale * (qn - E - thr_far);
                        const float Tf = tf - fabsf(tf) * (1.0f / 262144.0f) - 1e-30f;
                        const int nvb = min(64, lim - c0);
                        if (live) {
                            pr += nvb;  // counted far; the recorded ones are taken back below
                            p3 += nvb;
                        }
                        unsigned gm2 = 0;
#pragma unroll
                        for (int s = 0; s < 8; ++s) gm2 |= (live && m8[s] >= Tf ? 1u : 0u) << s;
                        unsigned gu2 = __reduce_or_sync(0xffffffffu, gm2);
                        while (gu2) {
                            const int s = __ffs(gu2) - 1;
                            gu2 &= gu2 - 1;
                            float x[8];
                            sm100::tmem_ld8(tmem + tb * kN + lane_base + c0 + 8 * s, x);
                            const bool take = (gm2 & (1u << s)) != 0;
                            const int g0 = c0 + 8 * s;
                            unsigned hit = 0;  // the group's elements that are not certainly far
#pragma unroll
                            for (int j = 0; j < 8; ++j) hit |= (take && x[j] >= Tf && g0 + j < lim ? 1u : 0u) << j;
                            const int nh = __popc(hit);
                            while (hit) {
                                const int j = __ffs(hit) - 1;
                                hit &= hit - 1;
                                if (rc < P.cap_rec) {
                                    rec[rc] = off + g0 + j;
                                    rdt[rc] = fmaf(-pick8(x, j), inv2s, qn);
                                }
                                ++rc;
                            }
                            pr -= nh;
                            p3 -= nh;
                            __syncwarp();
                        }
                    }
                }
                sm100::tc_fence_before();
                __syncwarp();
                if (lane == 0) sm100::mbar_arrive(&tempty[tb]);
                ++ti;
            }
            // U >= gamma_k^2 (U is an achieved k-th smallest upper bound)
            const float Uk = U;
            if (live && !(Uk < __int_as_float(0x7f800000))) fail = true;  // fewer than k candidates
#ifdef RBC_FAIL_WHY
            if (live && !(Uk < __int_as_float(0x7f800000))) atomicOr(P.fail + 1, 2);
            if (live && acoef == 0.0f) atomicOr(P.fail + 1, 4);
#endif
            const float ghi = sqrtf(Uk * kTie) * kUp;
            const float t9hi = 9.0f * ghi * ghi * (1.0f + kEps);

            // ---------- pass 2 (k > 1): count the far reps, record the rest with their estimate ----------
            for (int ch = 0; ch < (kSingle ? 0 : nchunks); ++ch) {
                const int off = ch * kN;
                const int lim = min(kN, static_cast<int>(P.nr) - off);
                const uint32_t tb = ti & 1;
                // reps with lb > max(9 ghi^2, (ghi + max psi of the chunk)^2) are pruned by both tests
                const float tpm = ghi + P.psimax[ch];
                const float thr_far = fmaxf(t9hi, tpm * tpm * (1.0f + kEps));
                // far  <=>  V < Tf   (Tf lowered by 2^-18 relative: only certain cases count as far)
                const float tf = 0.5f * scale * (qn - E - thr_far);
                const float Tf = tf - fabsf(tf) * (1.0f / 262144.0f) - 1e-30f;
                S1_WAIT(&tfull[tb], (ti >> 1) & 1, 9);
                sm100::tc_fence_after();
                for (int c0 = 0; c0 < S1_LIM(lim); c0 += 64) {
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
                    const int nvb = min(64, lim - c0);
                    if (live) {
                        pr += nvb;  // counted far; the recorded ones are taken back below
                        p3 += nvb;
                    }
                    float m8[8];
#pragma unroll
                    for (int s = 0; s < 8; ++s) m8[s] = max8(v + 8 * s);
                    unsigned gm = 0;
#pragma unroll
                    for (int s = 0; s < 8; ++s) gm |= (live && m8[s] >= Tf ? 1u : 0u) << s;
                    unsigned gu = __reduce_or_sync(0xffffffffu, gm);
                    while (gu) {
                        const int s = __ffs(gu) - 1;
                        gu &= gu - 1;
                        float x[8];
                        sm100::tmem_ld8(tmem + tb * kN + lane_base + c0 + 8 * s, x);
                        const bool take = (gm & (1u << s)) != 0;
                        const int g0 = c0 + 8 * s;
                        unsigned hit = 0;  // the group's elements that are not certainly far
#pragma unroll
                        for (int j = 0; j < 8; ++j) hit |= (take && x[j] >= Tf && g0 + j < lim ? 1u : 0u) << j;
                        const int nh = __popc(hit);
                        while (hit) {
                            const int j = __ffs(hit) - 1;
                            hit &= hit - 1;
                            if (rc < P.cap_rec) {
                                rec[rc] = off + g0 + j;
                                rdt[rc] = fmaf(-pick8(x, j), inv2s, qn);
                            }
                            ++rc;
                        }
                        pr -= nh;
                        p3 -= nh;
                        __syncwarp();
                    }
                }
                sm100::tc_fence_before();
                __syncwarp();
                if (lane == 0) sm100::mbar_arrive(&tempty[tb]);
                ++ti;
            }
            if (rc > P.cap_rec) fail = true;
#ifdef RBC_FAIL_WHY
            if (rc > P.cap_rec) atomicOr(P.fail + 1, 8);
#endif
            if (live) {
                // a failed row gets inert, in-range outputs: the batch is re-run on the
                // exact path, but the fix-up and stage 2 are already queued behind this kernel
                P.c1_cnt[qi] = fail ? -1 : count;
                P.c1_u[qi] = Uk * kTie;
                P.rec_e[qi] = E;
                P.pr[qi] = pr;
                P.p3[qi] = p3;
                P.rec_cnt[qi] = fail ? 0 : rc;
                if (fail) atomicExch(P.fail, 1);
            }
        }
    }
#ifdef RBC_S1_TIMING
    if (P.timing && lane == 0 && warp <= 2) {
        tw[12 + (warp == 2 ? 1 : 0)] = clock64() - t_start;  // wall of MMA / epilogue warp
        for (int j = 0; j < 14; ++j)
            if (tw[j]) atomicAdd(&P.timing[j], tw[j]);
    }
#endif
    sm100::tc_fence_before();
    __syncthreads();
    if (warp == 1) sm100::tmem_dealloc<256>(tmem);
}

// Distances of a query row (16 float4, zero padded to 64; shared memory,
// read as broadcasts) to a zero-padded 64-float row: padding terms are exact
// zeros, so summing all 64 coordinates reproduces the reference's d-term sum
// bit for bit.
__device__ __forceinline__ float exact_dist64(const float4 *__restrict__ qv, const float *__restrict__ row) {
    const float4 *r4 = reinterpret_cast<const float4 *>(row);
    double acc = 0.0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        float4 y[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) y[c] = __ldg(r4 + h * 8 + c);
#pragma unroll
        for (int c = 0; c < 8; ++c) acc = exact_acc4<RBC_L2>(acc, qv[h * 8 + c], y[c]);
    }
    return __double2float_rn(__dsqrt_rn(acc));
}

// Fix-up, one 8-lane group per query (4 queries per warp; queries in pilot
// order, so neighbouring groups share their reps in L1/L2), lanes over the
// query's entries: exact gamma_k and nearest rep from the gamma candidates
// (reference arithmetic, group top-k merge), exact decisions for the undecided
// reps, the 4 gamma cutoffs, the surviving segments (ascending rep position,
// ballot-compacted) and stats.  Eight lanes match the typical entry counts
// (a few gamma candidates, ~20 recorded reps), so few lanes idle.
#ifdef RBC_FIX_STATS
__device__ unsigned long long g_fix_stats[4];  // gamma exact, undecided exact, records, survivors
#endif
constexpr int kFixLanes = 8;
constexpr int kFixQueries = 32;  // queries per block (256 threads)

__device__ __forceinline__ uint64_t group_min_u64(uint64_t v) {
#pragma unroll
    for (int o = kFixLanes / 2; o > 0; o >>= 1) {
        const uint64_t w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w < v ? w : v;
    }
    return v;
}

#ifndef RBC_FIX_MB10
#define RBC_FIX_MB10 3
#endif
template <int KT>
__global__ void __launch_bounds__(kFixQueries * kFixLanes,
                                  KT == 1 ? 5 : (KT <= 8 ? 4 : (KT <= 10 ? RBC_FIX_MB10 : 2))) stage1_fixup_kernel(
    const float *__restrict__ q64, const int32_t *__restrict__ qorder, const float *__restrict__ reps64, int64_t nq,
    int k, const float *__restrict__ radii, const int64_t *__restrict__ offsets, const float *__restrict__ list_dists,
    const float *__restrict__ lskip, const float *__restrict__ c1_lb, const int32_t *__restrict__ c1_p, int cap1,
    const int32_t *__restrict__ c1_cnt, const float *__restrict__ c1_u, const int32_t *__restrict__ rec_cnt,
    const int32_t *__restrict__ rec, const float *__restrict__ rec_dt, const float *__restrict__ rec_e, int cap_rec,
    const int32_t *__restrict__ pr_in, const int32_t *__restrict__ p3_in, float *__restrict__ gamma_out, int32_t *__restrict__ nseg, int64_t *__restrict__ cand, int64_t *__restrict__ seg_off,
    int64_t *__restrict__ seg_start, int32_t *__restrict__ seg_len, int32_t *__restrict__ seg_list,
    float *__restrict__ seg_d1, uint64_t *__restrict__ order_key, int32_t *__restrict__ pr_out,
    int32_t *__restrict__ p3_out, int32_t *__restrict__ fail) {
    __shared__ float4 s_q[kFixQueries][16];
    const int lane = threadIdx.x & 31, sub = lane & (kFixLanes - 1);
    const int gq = threadIdx.x / kFixLanes;  // query slot in the block
    const int gshift = (lane / kFixLanes) * kFixLanes;
    const int64_t t = blockIdx.x * static_cast<int64_t>(kFixQueries) + gq;
    if (blockIdx.x * static_cast<int64_t>(kFixQueries) + (threadIdx.x & ~31) / kFixLanes >= nq) return;  // whole warp idle
    const bool live = t < nq;
    const int64_t i = live ? qorder[t] : 0;
    const int n1 = live ? c1_cnt[i] : -1;
    const int64_t base = i * static_cast<int64_t>(cap_rec);
    bool ok = n1 >= 0;  // a failed row (the batch is recomputed) gets inert outputs
    if (ok) {
        for (int c = sub; c < 16; c += kFixLanes) s_q[gq][c] = __ldg(reinterpret_cast<const float4 *>(q64 + i * 64) + c);
    }
    __syncwarp();
    const float4 *qv = s_q[gq];
    const float4 qa = qv[sub], qb = qv[sub + kFixLanes];  // this lane's 8 query coordinates
    // exact distance (reference arithmetic) for the lanes with `need`, one rep row at a time
    // per group: each of the 8 lanes sums 8 of the 64 fp64 reference terms (identical terms,
    // only the association differs), a shuffle tree adds the partials, and the fp32 result is
    // the reference's unless the tree sum's square root lies within 2^-44 (relative) of an fp32
    // rounding midpoint -- the sequential and tree sums differ by at most 2 * 63 * 2^-53
    // relative -- in which case the owner lane recomputes the sequential sum.
    auto coop_sq64 = [&](bool need, int32_t p) -> double {
        double res = 0.0;
        unsigned gm = (__ballot_sync(0xffffffffu, need) >> gshift) & ((1u << kFixLanes) - 1u);
        const int cnt = __popc(gm);
        const int mx = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(cnt));
        for (int t = 0; t < mx; ++t) {
            const int src = gm ? __ffs(gm) - 1 : 0;
            gm &= gm - 1;
            const int32_t pp = __shfl_sync(0xffffffffu, p, gshift + src);
            double part = 0.0;
            if (t < cnt) {
                const float4 *r4 = reinterpret_cast<const float4 *>(reps64 + static_cast<int64_t>(pp) * 64);
                const float4 ya = __ldg(r4 + sub), yb = __ldg(r4 + sub + kFixLanes);
                const float xs[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
                const float ys[8] = {ya.x, ya.y, ya.z, ya.w, yb.x, yb.y, yb.z, yb.w};
#pragma unroll
                for (int u = 0; u < 8; ++u) part = __dadd_rn(part, l2_term(xs[u], ys[u]));
            }
#pragma unroll
            for (int o = kFixLanes / 2; o > 0; o >>= 1) part = __dadd_rn(part, __shfl_xor_sync(0xffffffffu, part, o));
            if (t < cnt && sub == src) res = part;
        }
        return res;
    };
    // the reference's fp32 distance from a tree sum of its 64 terms (see coop_sq64): taken
    // unless the root lies within 2^-44 (relative) of an fp32 rounding midpoint, in which
    // case the sequential sum is recomputed
    auto verified = [&](double d2, int32_t p) -> float {
        const double r = __dsqrt_rn(d2);
        float f = __double2float_rn(r);
        const double mlo = 0.5 * (static_cast<double>(f) + static_cast<double>(nextafterf(f, -INFINITY)));
        const double mhi = 0.5 * (static_cast<double>(f) + static_cast<double>(nextafterf(f, INFINITY)));
        const double dl = 5.684341886080802e-14;  // 2^-44
        if (!(r * (1.0 - dl) > mlo && r * (1.0 + dl) < mhi))
            f = exact_dist64(qv, reps64 + static_cast<int64_t>(p) * 64);  // near a midpoint
        return f;
    };
    // ---- gamma_k over the candidates with lb <= U_k (lanes over candidates): the tree sums
    // (within 2^-45 of the sequential sums) of every candidate, then fp32 keys (verified
    // roots) only for the candidates within 2^-20 of the k-th smallest sum -- any other
    // candidate's distance exceeds the k nearest ones' by more than 2^-21 (relative), i.e.
    // by at least two fp32 ulps, so it cannot reach the k smallest keys (nor tie with them)
    const float ufin = ok ? c1_u[i] : 0.f;
    const int m1 = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(ok ? n1 : 0));
    double bd[KT];
    int32_t bp[KT];
#pragma unroll
    for (int j = 0; j < KT; ++j) {
        bd[j] = __longlong_as_double(0x7ff0000000000000ll);
        bp[j] = -1;
    }
    for (int e0 = 0; e0 < m1; e0 += kFixLanes) {
        const int e = e0 + sub;
        const bool pass = ok && e < n1 && c1_lb[i * cap1 + e] <= ufin;
        const int32_t p = pass ? c1_p[i * cap1 + e] : 0;
        const double d2 = coop_sq64(pass, p);
        if (pass) {
            double x = d2;
            int32_t y = p;
#pragma unroll
            for (int j = 0; j < KT; ++j) {  // sorted insert by (sum, position)
                const bool sw = x < bd[j] || (x == bd[j] && y < bp[j]);
                const double tx = sw ? bd[j] : x;
                const int32_t ty = sw ? bp[j] : y;
                if (sw) {
                    bd[j] = x;
                    bp[j] = y;
                }
                x = tx;
                y = ty;
            }
#ifdef RBC_FIX_STATS
            atomicAdd(&g_fix_stats[0], 1ull);
#endif
        }
    }
    double dk = __longlong_as_double(0x7ff0000000000000ll);  // >= the k-th smallest sum (ties pop together)
    {
        double cur[KT];
#pragma unroll
        for (int j = 0; j < KT; ++j) cur[j] = bd[j];
        for (int r = 0; r < k; ++r) {
            double m = cur[0];
#pragma unroll
            for (int o = kFixLanes / 2; o > 0; o >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
            dk = m;
            if (cur[0] == m) {
#pragma unroll
                for (int j = 0; j < KT - 1; ++j) cur[j] = cur[j + 1];
                cur[KT - 1] = __longlong_as_double(0x7ff0000000000000ll);
            }
        }
    }
    const double dthr = dk * (1.0 + 1.0 / 1048576.0);  // 2^-20
    uint64_t best[KT];
#pragma unroll
    for (int j = 0; j < KT; ++j) {
        best[j] = kEmptyKey;
        if (bp[j] >= 0 && bd[j] <= dthr) best[j] = pack_key(verified(bd[j], bp[j]), static_cast<uint32_t>(bp[j]));
    }
    // (ascending by sum and then position; the verified fp32 keys keep that order except
    // between equal fp32 values, so re-sort)
#pragma unroll
    for (int a = 1; a < KT; ++a)
#pragma unroll
        for (int b = a; b > 0; --b)
            if (best[b] < best[b - 1]) {
                const uint64_t t = best[b];
                best[b] = best[b - 1];
                best[b - 1] = t;
            }
    // group merge: the smallest key (nearest rep) and the k-th smallest (gamma_k)
    uint64_t first_key = kEmptyKey, kth = kEmptyKey;
    for (int r = 0; r < k; ++r) {
        const uint64_t m = group_min_u64(best[0]);
        if (r == 0) first_key = m;
        kth = m;
        if (best[0] == m && m != kEmptyKey) {  // keys are unique (distinct rep positions)
#pragma unroll
            for (int j = 0; j < KT - 1; ++j) best[j] = best[j + 1];
            best[KT - 1] = kEmptyKey;
        }
    }
    if (ok && kth == kEmptyKey) {  // cannot happen with a consistent bound; keep the result exact anyway
        if (sub == 0) atomicExch(fail, 1);
#ifdef RBC_FAIL_WHY
        if (sub == 0) atomicOr(fail + 1, 16);
#endif
        ok = false;
    }
    const float gf = ok ? key_dist(kth) : 0.f;
    const double g = gf, cutd = 4.0 * g;
    // ---- recorded reps: classify with the exact gamma on the interval [dt - E, dt + E]
    // (tri-state tests A: d > 3 gamma, B: d >= gamma + psi, C: d > gamma, search.py:62-74,
    // 194-195); only an undecided rep costs an exact distance
    const int n = ok ? rec_cnt[i] : 0;
    const int32_t *r = rec + base;
    const float *rd = rec_dt + base;
    const float E = ok ? rec_e[i] : 0.f;
    const float g2 = gf * gf, t9 = 9.0f * g2;
    int pr = 0, p3 = 0, ns = 0;
    long long cs = 0;
    unsigned first = 0xFFFFFFFFu;
    const int mn = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(n));
    for (int e0 = 0; e0 < mn; e0 += kFixLanes) {
        const int e = e0 + sub;
        bool emit = false;
        int32_t p = 0, len = 0;
        float dist = 0.f;
        if (e < n) {
            p = r[e];
            const float dt = rd[e];
            const float lb = dt - E, ub = dt + E;
            const float psi = radii[p];
            const float tp = gf + psi, tp2 = tp * tp;
            const bool a_t = lb > t9 * (1.0f + kEps), a_f = ub < t9 * (1.0f - kEps);
            const bool b_t = lb > tp2 * (1.0f + kEps), b_f = ub < tp2 * (1.0f - kEps);
            const bool c_t = lb > g2 * (1.0f + kEps), c_f = ub < g2 * (1.0f - kEps);
            const bool bc_t = b_t && c_t, bc_f = b_f || c_f;
            const float *row = reps64 + static_cast<int64_t>(p) * 64;
            bool surv;
            if ((a_t || a_f) && (bc_t || bc_f)) {
                p3 += a_t ? 1 : 0;
                pr += bc_t ? 1 : 0;
                surv = a_f && bc_f;
                // an upper bound of |q - r| (stage 2 only takes its operand scale from it and
                // computes |q - r|^2 itself in the A-operand prep)
                dist = surv ? sqrtf(fmaxf(ub, 0.f)) : 0.f;
            } else {
                dist = exact_dist64(qv, row);
#ifdef RBC_FIX_STATS
                atomicAdd(&g_fix_stats[1], 1ull);
#endif
                pr += pruned_radius(dist, psi, g) ? 1 : 0;
                p3 += pruned_3gamma(dist, g) ? 1 : 0;
                surv = survives(dist, psi, g);
            }
#ifdef RBC_FIX_STATS
            atomicAdd(&g_fix_stats[2], 1ull);
            if (surv) atomicAdd(&g_fix_stats[3], 1ull);
#endif
            if (surv) {
                const int32_t full = static_cast<int32_t>(offsets[p + 1] - offsets[p]);
                // the list's last (largest) distance is psi: the whole list is within 4 gamma iff psi <= 4 gamma
                len = static_cast<double>(psi) <= cutd
                          ? full
                          : list_cutoff_skip(list_dists + offsets[p], full, lskip + static_cast<int64_t>(p) * 32, cutd);
                emit = len > 0;
            }
        }
        const unsigned m = (__ballot_sync(0xffffffffu, emit) >> gshift) & ((1u << kFixLanes) - 1u);
        if (emit) {
            const int64_t at = base + ns + __popc(m & ((1u << sub) - 1u));
            seg_start[at] = offsets[p];
            seg_len[at] = len;
            seg_list[at] = p;
            seg_d1[at] = dist;
            cs += len;
            first = min(first, static_cast<unsigned>(p));
        }
        ns += __popc(m);
    }
#pragma unroll
    for (int o = kFixLanes / 2; o > 0; o >>= 1) {
        pr += __shfl_xor_sync(0xffffffffu, pr, o);
        p3 += __shfl_xor_sync(0xffffffffu, p3, o);
        cs += __shfl_xor_sync(0xffffffffu, cs, o);
        first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
    }
    if (live && sub == 0) {
        gamma_out[i] = gf;
        seg_off[i] = base;
        if (!ok) {
            nseg[i] = 0;
            cand[i] = 0;
            order_key[i] = 0;
        } else {
            if (pr_out) pr_out[i] = pr_in[i] + pr;
            if (p3_out) p3_out[i] = p3_in[i] + p3;
            nseg[i] = ns;
            cand[i] = cs;
            order_key[i] = (static_cast<uint64_t>(first & 0xFFFFFFu) << 24) | (key_id(first_key) & 0xFFFFFFu);
        }
    }
}

// dynamic shared memory: stages, A buffers, radii[nr], reduction slots, barriers
inline size_t s1_smem_bytes(int64_t nr) {
    return 1024 + kStages * kStageBytes + 2 * kABytes + (((nr + 3) & ~int64_t(3)) + 4) * sizeof(float) + 256;
}

}  // namespace

int tc1_index_prepare(rbc_index *idx, cudaStream_t st) {
    if (idx->kind != 0 || idx->metric != RBC_L2 || idx->d > 64 || idx->nr > kMaxRepsSmem) return RBC_OK;
    if (!tc_range_ok(idx->reps, idx->nr * idx->d, st)) return RBC_OK;  // (queries: pilot_key_kernel)
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
              cudaMalloc(&t->reps64, idx->nr * 64 * sizeof(float)) == cudaSuccess &&
              cudaMalloc(&t->pilots, kPilots * sizeof(int32_t)) == cudaSuccess &&
              cudaMalloc(&t->prow, kPilots * 8 * sizeof(uint4)) == cudaSuccess &&
              cudaMalloc(&t->pnorm, kPilots * sizeof(float)) == cudaSuccess &&
              cudaMalloc(&rmax_bits, sizeof(unsigned)) == cudaSuccess;
    auto cleanup = [&](int rc) {
        cudaFree(t->rb);
        cudaFree(t->psimax);
        cudaFree(t->lskip);
        cudaFree(t->c64);
        cudaFree(t->stat);
        cudaFree(t->reps64);
        cudaFree(t->pilots);
        cudaFree(t->prow);
        cudaFree(t->pnorm);
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
    pad_reps64_kernel<<<grid_for(idx->nr * 64, 256), 256, 0, st>>>(idx->reps, idx->nr, idx->d, t->reps64);
    {
        const int npilot = static_cast<int>(idx->nr < kPilots ? idx->nr : kPilots);
        const size_t fsmem = sizeof(float) * idx->nr;
        cudaFuncSetAttribute(pilot_fps_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(fsmem));
        pilot_fps_kernel<<<1, 1024, fsmem, st>>>(t->reps64, idx->nr, npilot, t->pilots);
        pilot_rows_kernel<<<grid_for(npilot * 8, 256), 256, 0, st>>>(t->reps64, t->pilots, npilot, t->prow, t->pnorm);
    }
    note_launch(9);
    float stat[2] = {1.f, 0.f};
    if (cudaMemcpyAsync(stat, t->stat, sizeof(stat), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return cleanup(fail(RBC_ECUDA, "tc1 index kernels"));
    cudaFree(rmax_bits);
    rmax_bits = nullptr;
    t->sG = stat[0];
    t->rmax = stat[1];
    idx->bytes += nchunks * kStageBytes + 66 * sizeof(float) + idx->nr * (64 + 32) * sizeof(float);
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
    cudaFree(t->reps64);
    cudaFree(t->pilots);
    cudaFree(t->prow);
    cudaFree(t->pnorm);
    delete t;
    idx->tc1 = nullptr;
}

bool tc_stage1_supported(const rbc_index *idx, int k) { return idx->tc1 != nullptr && k <= 16; }

static int g_num_sms1 = 0;

// Fused stage 1 + pruning, stream-ordered.  *fail_dev becomes nonzero when some
// row exhausted a buffer (the caller then runs the exact path).
int tc_stage1(const rbc_index *idx, const float *q, int64_t nq, int k, PruneOut &out, int32_t *fail_dev,
              cudaStream_t st) {
    const Tc1Index *t = static_cast<const Tc1Index *>(idx->tc1);
    const int ntiles = static_cast<int>((nq + kRows - 1) / kRows);
    const int cap1 = 32 + 16 * k;
    // per-query record / segment rows: room for every representative (a query whose k-th
    // nearest rep lies far away keeps most reps within 3 gamma_k), a multiple of 4 entries
    // (16-byte aligned rows for the tile kernels); the caller bounds nq (fused_chunk_limit)
    const int cap_rec = static_cast<int>((idx->nr + 3) & ~int64_t(3));
    DevBuf<float> q64buf, c1_lb, c1_u, rec_dt, rec_e;
    DevBuf<int32_t> c1_p, c1_cnt, pr0, p30, rec_cnt, rec, flags;
    DevBuf<int32_t> &qorder = out.qorder;
    DevBuf<uint32_t> pkey;
    DevBuf<unsigned> phist;  // [kPilots] bucket sizes, [kPilots] claim cursors
    DevBuf<float> pd2;       // [nq] upper bound of |q - nearest pilot|^2 (k = 1 seed bound)
    const float *q64 = q;
    if (idx->d != 64 || (reinterpret_cast<uintptr_t>(q) & 15) != 0) {
        RBC_CHECK(q64buf.alloc(nq * 64, st));
        pad_rows64(q, nq, idx->d, q64buf.get(), st);
        q64 = q64buf.get();
    }
    // query order: counting sort by nearest pilot
    const int npilot = static_cast<int>(idx->nr < kPilots ? idx->nr : kPilots);
    RBC_CHECK(qorder.alloc(nq, st));
    RBC_CHECK(pkey.alloc(nq, st));
    RBC_CHECK(phist.alloc(2 * kPilots + 1, st));  // + the query range flag
    RBC_CUDA(cudaMemsetAsync(phist.get(), 0, (2 * kPilots + 1) * sizeof(unsigned), st));
    RBC_CHECK(pd2.alloc(nq, st));
    pilot_key_kernel<<<grid_for(nq, kPilotWarps * 16), kPilotWarps * 32, 0, st>>>(
        q64, nq, t->prow, t->pnorm, npilot, t->reps64, t->pilots, pkey.get(), phist.get(), pd2.get());
    RBC_LAUNCHED();
    RBC_CHECK(flags.alloc(2, st));
    RBC_CHECK(out.s2_total.alloc(1, st));
    pilot_scatter_kernel<<<grid_for(nq, 128), 128, 0, st>>>(pkey.get(), nq, npilot, phist.get(), phist.get() + kPilots,
                                                           qorder.get(), flags.get(), out.s2_total.get(), fail_dev);
    out.s2_total_zeroed = true;
    RBC_LAUNCHED();
    RBC_CHECK(c1_lb.alloc(nq * cap1, st));
    RBC_CHECK(c1_p.alloc(nq * cap1, st));
    RBC_CHECK(c1_cnt.alloc(nq, st));
    RBC_CHECK(c1_u.alloc(nq, st));
    RBC_CHECK(pr0.alloc(nq, st));
    RBC_CHECK(p30.alloc(nq, st));
    RBC_CHECK(rec_cnt.alloc(nq, st));
    RBC_CHECK(rec.alloc(nq * cap_rec, st));
    RBC_CHECK(rec_dt.alloc(nq * cap_rec, st));
    RBC_CHECK(rec_e.alloc(nq, st));
    RBC_CHECK(out.gamma.alloc(nq, st));
    RBC_CHECK(out.nseg.alloc(nq, st));
    RBC_CHECK(out.cand.alloc(nq, st));
    RBC_CHECK(out.seg_off.alloc(nq + 1, st));
    RBC_CHECK(out.order_key.alloc(nq, st));
    RBC_CHECK(out.seg_start.alloc(nq * cap_rec, st));
    RBC_CHECK(out.seg_len.alloc(nq * cap_rec, st));
    RBC_CHECK(out.seg_list.alloc(nq * cap_rec, st));
    RBC_CHECK(out.seg_d1.alloc(nq * cap_rec, st));
    S1Params P;
    P.rb = t->rb;
    P.plane1 = t->plane1 ? 1 : 0;
    P.nr = idx->nr;
    P.sG = t->sG;
    P.rmax = t->rmax;
    P.c64 = t->c64;
    P.psimax = t->psimax;
    P.pd2 = pd2.get();
    P.q64 = q64;
    P.qorder = qorder.get();
    P.radii = idx->radii;
    P.k = k;
    P.nq = nq;
    P.ntiles = ntiles;
    P.c1_lb = c1_lb.get();
    P.c1_p = c1_p.get();
    P.cap1 = cap1;
    P.c1_cnt = c1_cnt.get();
    P.c1_u = c1_u.get();
    P.pr = pr0.get();
    P.p3 = p30.get();
    P.rec_cnt = rec_cnt.get();
    P.rec = rec.get();
    P.rec_dt = rec_dt.get();
    P.rec_e = rec_e.get();
    P.cap_rec = cap_rec;
    P.fail = fail_dev;
    P.tile_counter = flags.get() + 1;
    if (g_num_sms1 == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms1, cudaDevAttrMultiProcessorCount, dev);
    }
    // persistent CTAs, two per SM when the representatives' radii fit (tiles come from a counter)
    const size_t smem = s1_smem_bytes(idx->nr);
    const int per_sm = smem <= 112 * 1024 ? 2 : 1;  // two CTAs (2 x 256 TMEM columns) when shared memory allows
    const unsigned grid = static_cast<unsigned>(ntiles < per_sm * g_num_sms1 ? ntiles : per_sm * g_num_sms1);
    auto launch = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        kern<<<grid, kThreads, smem, st>>>(P);
    };
    P.timing = nullptr;
#ifdef RBC_S1_TIMING
    DevBuf<unsigned long long> timing;
    if (getenv("RBC_DEBUG_S1")) {
        RBC_CHECK(timing.alloc(14, st));
        RBC_CUDA(cudaMemsetAsync(timing.get(), 0, sizeof(unsigned long long) * 14, st));
        P.timing = timing.get();
    }
#endif
    if (k == 1) launch(stage1_tc_kernel<1>);
    else if (k <= 4) launch(stage1_tc_kernel<4>);
    else if (k <= 8) launch(stage1_tc_kernel<8>);
    else if (k == 10) launch(stage1_tc_kernel<10>);  // the k of cfg3/cfg5: no k-th select
    else launch(stage1_tc_kernel<16>);
    RBC_LAUNCHED();
#ifdef RBC_S1_TIMING
    if (P.timing) {
        unsigned long long h[14];
        cudaMemcpy(h, P.timing, sizeof(h), cudaMemcpyDeviceToHost);
        const char *nm[14] = {"prod:tile_empty", "prod:empty", "mma:tile_full", "mma:afull", "mma:full", "mma:tempty",
                              "epi:tile_full", "epi:aempty", "epi:tfull1", "epi:tfull2", "epi:qfull", "-",
                              "wall:prod+mma", "wall:epi"};
        fprintf(stderr, "[s1] per-CTA cycles (grid %u):", grid);
        for (int j = 0; j < 14; ++j) fprintf(stderr, " %s=%.0f", nm[j], double(h[j]) / grid);
        fprintf(stderr, "\n");
    }
#endif
    const unsigned fgrid = grid_for(nq, kFixQueries);
#define RBC_FIXUP(KT)                                                                                                 \
    stage1_fixup_kernel<KT><<<fgrid, kFixQueries * kFixLanes, 0, st>>>(                                                           \
        q64, qorder.get(), t->reps64, nq, k, idx->radii, idx->offsets, idx->list_dists, t->lskip, c1_lb.get(),          \
        c1_p.get(),                                                                                                    \
        cap1, c1_cnt.get(), c1_u.get(), rec_cnt.get(), rec.get(), rec_dt.get(), rec_e.get(), cap_rec, pr0.get(),        \
        p30.get(), out.gamma.get(),                                                                                    \
        out.nseg.get(), out.cand.get(), out.seg_off.get(), out.seg_start.get(), out.seg_len.get(), out.seg_list.get(), \
        out.seg_d1.get(), out.order_key.get(), out.pr, out.p3, fail_dev)
    if (k == 1) RBC_FIXUP(1);
    else if (k <= 4) RBC_FIXUP(4);
    else if (k <= 8) RBC_FIXUP(8);
    else if (k == 10) RBC_FIXUP(10);
    else RBC_FIXUP(16);
#undef RBC_FIXUP
    RBC_LAUNCHED();
#ifdef RBC_FIX_STATS
    if (getenv("RBC_DEBUG_S1")) {
        unsigned long long h[4];
        cudaMemcpyFromSymbol(h, g_fix_stats, sizeof(h));
        const unsigned long long z[4] = {0, 0, 0, 0};
        cudaMemcpyToSymbol(g_fix_stats, z, sizeof(z));
        fprintf(stderr, "[fixup] per query: gamma exact %.2f, undecided exact %.2f, records %.2f, survivors %.2f\n",
                double(h[0]) / nq, double(h[1]) / nq, double(h[2]) / nq, double(h[3]) / nq);
    }
#endif
    return RBC_OK;
}

}  // namespace rbc
