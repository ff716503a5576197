// tc_stage2.cu -- exact-search stage 2 on the 5th-generation tensor cores.
//
// Work unit: a TILE of 128 queries that share (mostly) the same surviving
// ownership lists (queries are grouped by (first surviving list, nearest
// rep)).  For every list p in the union of the tile's survivors, and every
// 256-row chunk of p's scanned prefix:
//
//   A_p = f16((q_i - r_p) * sA)   128 x 64 (+16), K-major, built by 4 "prep" warps
//   B   = f16((x_j - r_p) * sB_p) N x 64 (+16) rows, pre-swizzled in HBM, cp.async.bulk per chunk
//   D   = A_p . B^T               tcgen05.mma kind::f16 into TMEM (fp32), double-buffered
//
// Centering both operands on the list's representative keeps |a|,|b| at the
// scale of the query->rep and point->rep distances, so the expanded form
//   d^2 = |q - r_p|^2 + |x - r_p|^2 - 2 (q - r_p).(x - r_p)
// (the first term is stage 1's exact distance) has a rigorous error bound
//   E <= C1 |a||b| + C2 (|a|^2 + |b|^2) + C4 |b| / sA
// small enough that only a handful of points per query need the exact
// re-rank.  The per-column term |x - r_p|^2 / 2 is folded into the MMA as
// two extra K columns (hi/lo f16 split; A side = -sA/sB), so the
// accumulator is directly V = sA sB ((q-r).(x-r) - |x-r|^2/2), and
//   lb = |q - r_p|^2 - E - 2 V / (sA sB)  <=  d^2  <=  lb + 2E.
// The epilogue (4 warps, one TMEM lane = one query row per thread) reduces
// each 32-column chunk to its maximum V (3-input FMNMX), updates the row's
// running best upper bound from it (k = 1) and only drops to the slow path
// when some element can still beat the k-th best; there candidates are
// appended to a per-query buffer.  A separate kernel then re-ranks every
// buffered candidate with the reference's exact fp64 arithmetic
// (common.cuh exact_dist) and emits key64 = (f32 dist, id), so results are
// bit-identical to the reference.  A query whose buffer overflows is
// recomputed by the exact SIMT scan.
//
// Roles (320 threads, 1 CTA per SM, persistent, no CTA-wide barrier in the
// steady state; tiles come from an LPT-ordered global queue through a
// 2-slot shared-memory ring):
//   warp 0      scheduler + producer: cp.async.bulk of B chunks, 4-stage ring
//   warp 1      MMA issuer + TMEM owner (512 columns = 2 x 256 fp32 accumulators)
//   warps 2..9  epilogue, two warps per TMEM lane quadrant (one per 128-column
//               half of each chunk): A-operand prep for the next list (each warp
//               its half of K), candidate filter, per-half candidate buffers
#include <cub/cub.cuh>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "index.cuh"
#include "kernels.cuh"
#include "search.cuh"
#include "sm100.cuh"
#include "tc_scan.cuh"

namespace rbc {

namespace {

constexpr int kRows = 128;       // queries per tile = UMMA M = TMEM lanes
constexpr int kNmax = 256;       // largest UMMA N per chunk (N = 256 keeps the single MMA thread compute-bound)
constexpr int kParts = 2;        // epilogue warps per TMEM lane quadrant (column halves / K halves)
constexpr int kEpiWarps = 4 * kParts;
// warp group 0: producer (warp 0), MMA issuer (warp 1), two idle warps; warp groups 1-2: the
// epilogue.  Launched at 168 registers per thread (384 threads, 1 CTA/SM); warp group 0 gives
// registers back (setmaxnreg.dec to kRegsCtl) and the epilogue takes them (setmaxnreg.inc to
// kRegsEpi) so two TMEM loads can be in flight per epilogue thread without spills.  Per SMSP:
// warps {w, w + 4, w + 8} hold kRegsCtl + 2 kRegsEpi <= 512 registers per lane.
constexpr int kEpiWarp0 = 4;
constexpr int kThreads = 32 * kEpiWarp0 + 32 * kEpiWarps;
constexpr int kRegsCtl = 56;
constexpr int kRegsEpi = 224;
static_assert(kRegsCtl + 2 * kRegsEpi <= 512, "per-SMSP register file");
constexpr int kTailRows = kNmax; // zero rows after the last list (bulk copies may overrun)
constexpr int kP0 = 128;         // plane-0 row bytes: 64 f16, SWIZZLE_128B
constexpr int kP1 = 32;          // plane-1 row bytes: 16 f16, SWIZZLE_32B (aug columns when d > 62)
constexpr int kLSlots = 4;       // per-list data ring slots
constexpr int kMaxSplit = 4;     // k > 1: a heavy tile's work items are split over up to 4 CTAs
constexpr int kMaxSlots = kParts * kMaxSplit;  // candidate slots per query (column parts x splits)
// Per K-plane count NP (d <= 64 * NP): NP = 1 for d <= 64; NP = 2 for d <= 128 (two SW128
// planes, 128-column chunks and a 3-stage ring so the A/B buffers fit in shared memory).
template <int NP>
struct S2Cfg {
#ifndef RBC_S2_N1
#define RBC_S2_N1 256
#endif
#ifndef RBC_S2_ACC2
#define RBC_S2_ACC2 4
#endif
    static constexpr int kN = NP == 1 ? RBC_S2_N1 : 128;  // UMMA N per chunk
    static constexpr int kAcc = NP == 1 ? 512 / RBC_S2_N1 : RBC_S2_ACC2;  // TMEM accumulator stages
    static constexpr int kStages = 3 * 256 / kN / NP;     // B ring depth (B traffic is not the bound)
    static constexpr int kCols = kN / kParts;        // columns of each chunk per epilogue warp
    static constexpr int kKd = 64 * NP / kParts;     // A-operand dims per epilogue warp
    static constexpr int kStageBytes = kN * (NP * kP0 + kP1);
    static constexpr int kABytes = kRows * (NP * kP0 + kP1);
    static constexpr int kTmemCols = kAcc * kN;      // kAcc accumulators
    // per-list data ring (work item + representative row + its B rounding error), staged by the
    // producer one list ahead so no role waits on a dependent global load at a list switch
    static constexpr int kRepStride = 64 * NP + 4;                        // floats per rep row
    static constexpr int kLSlotBytes = 32 + kRepStride * 4 + kRows * 4;  // WorkItem + rep row + row cutoffs
    // NP = 1: the tile's query rows in shared memory (the A-operand preparation reads them per
    // list; registers go to two TMEM loads in flight instead), stride 68 floats (conflict-free
    // 16-byte loads of 32 consecutive rows)
    static constexpr int kQStride = 68;
    static constexpr int kQSmemFloats = NP == 1 ? kRows * kQStride : 0;
    static constexpr size_t kSmem = 1024 + kStages * kStageBytes + 2 * kABytes +
                                    (kEpiWarps * kCols + 8 * kParts * kRows + kQSmemFloats) * sizeof(float) +
                                    kLSlots * kLSlotBytes + 512;
};

// error-bound constants (factor-2 safety on each term; K <= 80 accumulated products)
constexpr float kC1 = 4.0f * (1.0f / 1024.0f + 128.0f / 4194304.0f);  // f16 rounding of a and b, fp32 accumulate
#ifdef RBC_S2_NOHOLD
constexpr bool kHold = false;  // diagnostic variant
#else
constexpr bool kHold = true;   // k = 1: newest qualifying group held in registers
#endif
constexpr float kAccErr = 4.0f * 128.0f / 4194304.0f;                  // fp32 accumulation share of kC1 (K <= 80;
                                                                       // doubled for the K <= 144 of NP = 2)
constexpr float kC2 = 1.0f / 1048576.0f;                              // norms, aug split, epilogue rounding
constexpr float kC4 = 1.0f / 262144.0f;                               // f16 subnormal flush (absolute, scaled)
constexpr float kUp = 1.0f + 1.0f / 1048576.0f;                       // rounding-up factor for norms
constexpr float kTie = 1.0f + 1.0f / 524288.0f;                       // tie slack: 8 fp32 ulps of the distance
constexpr float kD1 = 1.0f / 32768.0f;                                // approximate stage-1 distance (A2 term)
constexpr float kUq = 1.0f + 1.0f / 65536.0f;                          // ... and its |a| bound

struct TcIndex {
    int64_t npad = 0;
    int np = 1;               // 64-wide K planes (d <= 64 np)
    int64_t rows = 0;         // rows per plane (npad + tail)
    bool plane1 = false;      // aug columns in a separate 16-wide plane (d > 64 np - 2)
    uint8_t *xh0 = nullptr;   // [np][rows][128 B] f16 residual rows (+aug in the last plane when d <= 64 np - 2), SW128
    uint8_t *xh1 = nullptr;   // [npad + tail][32 B] aug plane, SW32 pre-swizzled (d > 62 only)
    float *gcol = nullptr;    // [npad + tail] (|x - r_p|^2 / 2) * sB_p (fallback when -sA/sB is not an f16 normal)
    int64_t *poff = nullptr;  // [nr + 1] padded (8-row aligned) list offsets
    float *sB = nullptr;      // [nr] per-list power-of-two scale
    float *dbmax = nullptr;   // [nr] max over the list of |b - f16(b)| (scaled residual rows, f16 rounding)
    float *reps64 = nullptr;  // [nr][64 np + 4] representatives, zero padded; [64 np] = dbmax[p]
};

// one (tile, list) work item, 32 bytes
struct __align__(16) WorkItem {
    int32_t p;       // list (rep position)
    int32_t ext;     // scanned prefix: max cutoff over the tile's rows
    float sA;        // A scale (power of two)
    float sB;        // B scale of the list
    float radius;    // list radius psi_p
    float aug;       // A-side folded-norm coefficient -sA/sB (0 = subtract in the epilogue)
    int32_t poff;    // padded row offset of the list in xh0/xh1/gcol
    int32_t csr;     // CSR offset of the list (positions into xp / perm)
};

struct S2Params {
    const uint8_t *xh0;
    int64_t plane_bytes;        // byte stride between the K planes of xh0
    const uint8_t *xh1;
    const float *gcol;
    const float *reps64;
    const float *dbmax;         // [nr] per-list max f16 rounding error of the B rows (scaled)
    int plane1;
    const float *q64;           // queries, rows padded to 64 NP floats
    const float *gamma;         // [nq] gamma_k
    int k;
    int ntiles;
    const int32_t *tile_order;  // LPT order
    const int4 *vt;             // virtual tiles {tile, first work item, end, split} in LPT order (nullptr: whole tiles)
    const int32_t *nvt;         // their count (device)
    int nslot;                  // candidate slots per query: kParts x splits
    const int32_t *order;       // query order: tile t holds order[128 t .. 128 t + 127] (nq entries)
    int64_t nq;
    const int64_t *work_off;    // [ntiles] first work item of each tile
    const int64_t *nwork;       // [ntiles] its work items
    const unsigned long long *work_total;
    const WorkItem *work;       // [total work]
    const int32_t *cut;         // [total work][128] per-row cutoff (0 = list not a survivor for the row);
                                // null: every row scans the item's whole prefix (brute force)
    float *cand_lb;
    int32_t *cand_pos;
    int cap;
    int32_t *cand_count;        // [nq][nslot] buffered groups, -1 = overflow
    float *cand_ufin;           // [nq][nslot] final k-th best upper bound (with tie slack)
    int32_t *overflow_list;
    int32_t *overflow_count;
    int32_t *tile_counter;
    int64_t cap_work;
    unsigned long long *timing;  // diagnostic [grid][8] role wait/busy cycles (nullptr = off)
};

__device__ __forceinline__ int roundup16(int x) { return (x + 15) & ~15; }

constexpr int kSegBatch = 8;  // per-row segment entries loaded together in the tile kernels
#ifndef RBC_FILL_WAYS
#define RBC_FILL_WAYS 4
#endif
constexpr int kFillWays = RBC_FILL_WAYS;          // tile_fill_kernel threads per row
constexpr int kFillThreads = kFillWays * kRows;

// Entries a[s .. s + min(rem, 8)) of a 32-bit array (the rest = fill): 16-byte vector
// loads where the address is aligned and the quad lies inside the row, so a thread
// reading its own row costs one L1 wavefront per four entries instead of one per entry.
__device__ __forceinline__ void load8_u32(const uint32_t *__restrict__ a, int64_t s, int rem, uint32_t (&o)[8],
                                          uint32_t fill) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int b = 4 * h;
        if (rem >= b + 4 && ((s + b) & 3) == 0) {
            const uint4 v = __ldg(reinterpret_cast<const uint4 *>(a + s + b));
            o[b] = v.x;
            o[b + 1] = v.y;
            o[b + 2] = v.z;
            o[b + 3] = v.w;
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) o[b + j] = b + j < rem ? __ldg(a + s + b + j) : fill;
        }
    }
}

// Diagnostic role timing (build with -DRBC_S2_TIMING and run with RBC_DEBUG_S2=1):
// cycles each role spends waiting on its mbarriers, per CTA.
#ifdef RBC_S2_TIMING
__device__ __forceinline__ void mbar_wait_t(uint64_t *bar, uint32_t parity, unsigned long long &acc) {
    const unsigned long long t0 = clock64();
    sm100::mbar_wait(bar, parity);
    acc += clock64() - t0;
}
#define S2_WAIT(bar, parity, slot) mbar_wait_t(bar, parity, tw[slot])
#define S2_TIME(stmt) stmt
#else
#define S2_WAIT(bar, parity, slot) sm100::mbar_wait(bar, parity)
#define S2_TIME(stmt)
#endif

__device__ __forceinline__ float max8(const float *v) { return sm100::max8(v); }

// ---- index preparation ----------------------------------------------------------
__global__ void list_scale_kernel(const float *__restrict__ radii, int64_t nr, float *__restrict__ sB) {
    const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (p >= nr) return;
    const float r = radii[p];
    int e = 0;
    if (r > 0.f) frexpf(r, &e);  // r = m * 2^e, m in [0.5, 1)  ->  r * 2^-e < 1
    sB[p] = r > 0.f ? ldexpf(1.0f, -e) : 1.0f;
}

// f16 residual rows of the lists (pre-swizzled), folded-norm columns, fallback column.
// Grid (list, row slice): blockIdx.x = list p, blockIdx.y strides over its rows, so a
// single long list (the brute-force scan) is prepared by many blocks.  dbmax[p] must be
// zero on entry (max over the row slices through a float-bits atomic).
__global__ void residual_rows_kernel(const float *__restrict__ xp, const float *__restrict__ reps,
                                     const int64_t *__restrict__ offsets, const int64_t *__restrict__ poff,
                                     const float *__restrict__ sB, int d, int np, int64_t plane_bytes, int plane1,
                                     uint8_t *__restrict__ xh0,
                                     uint8_t *__restrict__ xh1, float *__restrict__ gcol, float *__restrict__ dbmax) {
    __shared__ unsigned s_db;
    if (threadIdx.x == 0) s_db = 0;
    __syncthreads();
    const int64_t p = blockIdx.x;
    const int64_t len = offsets[p + 1] - offsets[p];
    const float s = sB[p];
    const float *r = reps + p * d;
    for (int64_t j = blockIdx.y * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < len;
         j += static_cast<int64_t>(gridDim.y) * blockDim.x) {
        const float *x = xp + (offsets[p] + j) * d;
        const int64_t row = poff[p] + j;
        double h = 0.0;
        for (int k = 0; k < d; ++k) {
            const double b = __fsub_rn(x[k], r[k]);
            h += b * b;
        }
        const float hf = static_cast<float>(h);
        const float gp = hf * 0.5f * s * s;  // (|b|^2 / 2) sB^2, < 0.5
        const __half ghi = __float2half_rn(gp);
        const __half glo = __float2half_rn(gp - __half2float(ghi));
        const uint32_t aug = static_cast<uint32_t>(__half_as_ushort(ghi)) |
                             (static_cast<uint32_t>(__half_as_ushort(glo)) << 16);
        float db2 = 0.f;  // |b - f16(b)|^2 of this row (scaled units)
        for (int c = 0; c < 8 * np; ++c) {
            uint8_t *dst = xh0 + (c >> 3) * plane_bytes + row * kP0;
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int k0 = c * 8 + 2 * e, k1 = k0 + 1;
                const float b0 = k0 < d ? __fsub_rn(x[k0], r[k0]) : 0.f;
                const float b1 = k1 < d ? __fsub_rn(x[k1], r[k1]) : 0.f;
                w[e] = sm100::pack_f16x2_sat(b0 * s, b1 * s);
                __half2 h;
                *reinterpret_cast<uint32_t *>(&h) = w[e];
                const float2 hf2 = __half22float2(h);
                const float e0 = b0 * s - hf2.x, e1 = b1 * s - hf2.y;
                db2 = fmaf(e0, e0, fmaf(e1, e1, db2));
            }
            if (!plane1 && c == 8 * np - 1) w[3] = aug;  // last two columns of the last plane
            *reinterpret_cast<uint4 *>(dst + (((c & 7) ^ (row & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        if (plane1) {
            uint8_t *d1p = xh1 + row * kP1;
            const int sw = static_cast<int>((row >> 2) & 1);
            *reinterpret_cast<uint4 *>(d1p + ((0 ^ sw) << 4)) = make_uint4(aug, 0, 0, 0);
            *reinterpret_cast<uint4 *>(d1p + ((1 ^ sw) << 4)) = make_uint4(0, 0, 0, 0);
        }
        gcol[row] = hf * 0.5f * s;
        atomicMax(&s_db, __float_as_uint(sqrtf(db2)));
    }
    __syncthreads();
    if (threadIdx.x == 0 && s_db) atomicMax(reinterpret_cast<unsigned *>(dbmax) + p, s_db);
}

__global__ void rep_dbmax_kernel(const float *__restrict__ dbmax, int64_t nr, int stride, float *__restrict__ reps) {
    const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (p < nr) reps[p * stride + stride - 4] = dbmax[p];
}

// rows of src [rows][d] -> dst [rows][w], zero padded (w = 64, 128, or those + 4)
__global__ void pad64_rows_kernel(const float *__restrict__ src, int64_t rows, int d, float *__restrict__ dst,
                                  int w = 64) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t >= rows * w) return;
    const int64_t r = t / w;
    const int c = static_cast<int>(t - r * w);
    dst[t] = c < d ? src[r * d + c] : 0.f;
}

// ---- tile preparation -----------------------------------------------------------------
// query grouping key (first surviving list, nearest rep) packed into 2 * kb bits, so the
// sort runs ceil(2 kb / 8) radix passes instead of six, plus the identity payload
__global__ void group_key_kernel(const uint64_t *__restrict__ order_key, int64_t nq, int kb, uint32_t *__restrict__ key,
                                 int32_t *__restrict__ ids) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t >= nq) return;
    const uint64_t o = order_key[t];
    const uint32_t mask = (1u << kb) - 1u;
    key[t] = ((static_cast<uint32_t>(o >> 24) & mask) << kb) | (static_cast<uint32_t>(o) & mask);
    ids[t] = static_cast<int32_t>(t);
}

// union of the tile's surviving lists: work items, per-row cutoffs and stage-1
// distances, and the tile's total work (for the LPT order)
__global__ void __launch_bounds__(kFillThreads) tile_fill_kernel(
    const int32_t *__restrict__ order, int64_t nq, int64_t *__restrict__ nwork, int64_t *__restrict__ work_off,
    unsigned long long *__restrict__ work_total, int32_t *__restrict__ tile_ids, const int64_t *__restrict__ seg_off, const int32_t *__restrict__ seg_cnt,
    const int32_t *__restrict__ seg_list, const int32_t *__restrict__ seg_len, const float *__restrict__ seg_d1,
    const uint64_t *__restrict__ order_key,
    int64_t nr, const float *__restrict__ sB, const float *__restrict__ radii, const int64_t *__restrict__ poff,
    const int64_t *__restrict__ offsets, WorkItem *__restrict__ work,
    int32_t *__restrict__ cut, uint64_t *__restrict__ tile_key, int warm,
    int64_t cap_work, int32_t *__restrict__ cand_count, int nslot, int32_t *__restrict__ counters) {
    if (threadIdx.x == 0) tile_ids[blockIdx.x] = static_cast<int32_t>(blockIdx.x);
    extern __shared__ int32_t sm[];
    int32_t *maxlen = sm;           // [nr]
    int32_t *maxd1 = sm + nr;       // [nr] float bits (non-negative)
    int32_t *nearcnt = sm + 2 * nr; // [nr]
    typedef cub::BlockScan<int, kFillThreads> Scan;
    // kFillWays threads per row: `way` takes every kFillWays-th batch of the row's segments
    const int row = threadIdx.x & (kRows - 1), way = threadIdx.x / kRows;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ unsigned long long s_work, s_off;
    __shared__ int s_lists;
    for (int64_t p = threadIdx.x; p < nr; p += blockDim.x) maxlen[p] = maxd1[p] = nearcnt[p] = 0;
    if (threadIdx.x == 0) {
        s_work = 0;
        s_lists = 0;
    }
    __syncthreads();
    const int64_t tq = static_cast<int64_t>(blockIdx.x) * kRows + row;
    // stage 2's per-query group counts and its two counters start at zero (in place of two
    // memset nodes; unconditional: the re-rank reads the counts even when stage 2 bails out)
    if (tq < nq)
        for (int h = way; h < nslot; h += kFillWays) cand_count[nslot * tq + h] = 0;
    if (blockIdx.x == 0 && threadIdx.x < 2) counters[threadIdx.x] = 0;
    const int32_t qi = tq < nq ? order[tq] : -1;
    const int64_t s0 = qi >= 0 ? seg_off[qi] : 0;
    const int cnt = qi >= 0 ? seg_cnt[qi] : 0;
    {
        // shared-memory max atomics, warp-aggregated when all 32 rows hold the same list at
        // this step (common at k = 1: segments ascend by list and the rows share lists).
        // Each row's segments are read kSegBatch at a time (independent loads in flight).
        const int lane = threadIdx.x & 31;
        const int wmax = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(cnt));
        for (int it0 = way * kSegBatch; it0 < wmax; it0 += kFillWays * kSegBatch) {
            uint32_t pu[kSegBatch], lb[kSegBatch], db[kSegBatch];
            const int rem = max(cnt - it0, 0);
            load8_u32(reinterpret_cast<const uint32_t *>(seg_list), s0 + it0, rem, pu, 0xFFFFFFFFu);
            load8_u32(reinterpret_cast<const uint32_t *>(seg_len), s0 + it0, rem, lb, 0u);
            load8_u32(reinterpret_cast<const uint32_t *>(seg_d1), s0 + it0, rem, db, 0u);
#pragma unroll
            for (int j = 0; j < kSegBatch; ++j) {
                if (it0 + j >= wmax) break;  // warp-uniform
                const int32_t p = static_cast<int32_t>(pu[j]);
                // whole warp on one list: one full-mask reduction and one atomic pair.  Otherwise
                // every lane updates on its own (a partial-mask __reduce_max_sync is a loop over
                // the distinct masks: ~14 CREDUX per step when the rows' lists diverge, k > 1)
                int same;
                __match_all_sync(0xffffffffu, p, &same);
                if (same) {
                    const unsigned mlen = __reduce_max_sync(0xffffffffu, lb[j]), md1 = __reduce_max_sync(0xffffffffu, db[j]);
                    if (p >= 0 && lane == 0) {
                        atomicMax(&maxlen[p], static_cast<int>(mlen));
                        atomicMax(&maxd1[p], static_cast<int>(md1));
                    }
                } else if (p >= 0) {
                    atomicMax(&maxlen[p], static_cast<int>(lb[j]));
                    atomicMax(&maxd1[p], static_cast<int>(db[j]));
                }
            }
        }
        const int32_t nr_near = qi >= 0 ? static_cast<int32_t>(order_key[qi] & 0xFFFFFF) : -1;
        const unsigned grp = __match_any_sync(0xffffffffu, nr_near);
        if (way == 0 && qi >= 0 && lane == __ffs(grp) - 1) atomicAdd(&nearcnt[nr_near], __popc(grp));
    }
    __syncthreads();
    // one pass over this thread's contiguous range of lists: the tile's total work (LPT
    // key), its list count, the sort keys of the lists that are some row's nearest rep
    // ("F" lists, ordered first: most rows first, so each row's running bound tightens
    // early and fewer candidate groups are buffered) and the count of the others
    __shared__ unsigned long long s_fkey[kRows];
    __shared__ int s_nf;
    if (threadIdx.x == 0) s_nf = 0;
    __syncthreads();
    const int64_t per = (nr + kFillThreads - 1) / kFillThreads;
    const int64_t pa = threadIdx.x * per, pe = min(nr, pa + per);
    unsigned long long wsum = 0;
    int nl = 0, c = 0;
    for (int64_t p = pa; p < pe; ++p) {
        const int ml = maxlen[p];
        if (ml > 0) {
            wsum += ml;
            ++nl;
            if (nearcnt[p] > 0) {
                const int slot = atomicAdd(&s_nf, 1);  // <= 128 distinct nearest reps per tile
                s_fkey[slot] = (static_cast<unsigned long long>(kRows - nearcnt[p]) << 32) | static_cast<uint64_t>(p);
            } else {
                ++c;
            }
        }
    }
    atomicAdd(&s_work, wsum);
    atomicAdd(&s_lists, nl);
    int pos, total;
    Scan(scan_tmp).ExclusiveSum(c, pos, total);
    __syncthreads();
    // the tile claims its range of the shared work array with one atomic (an undersized
    // array makes the tiles that do not fit skip their writes; stage 2 then bails out and
    // the caller re-runs)
    if (threadIdx.x == 0) {
        const int64_t nw = s_lists + (warm && s_lists > 0 ? 1 : 0);
        s_off = atomicAdd(work_total, static_cast<unsigned long long>(nw));
        nwork[blockIdx.x] = nw;
        work_off[blockIdx.x] = static_cast<int64_t>(s_off);
    }
    __syncthreads();
    // with warm-up, slot w0 is a max-only copy of the first list (k = 1: it
    // tightens the running bound before any candidate is buffered)
    const int64_t wbase = static_cast<int64_t>(s_off), wn = nwork[blockIdx.x];
    if (wbase + wn > cap_work) return;  // capacity exceeded: the caller re-runs with the exact size
    const int64_t w0 = wbase + ((warm && wn > 0) ? 1 : 0);
    // zero this thread's cutoff column of the tile's work items (its own later writes win)
    for (int64_t w = wbase + way; w < wbase + wn; w += kFillWays) cut[w * kRows + row] = 0;
    // positions (nearcnt is reused as list -> work index): F lists by rank, then the others
    const int nf = s_nf;
    for (int64_t p = pa; p < pe; ++p)
        if (maxlen[p] > 0 && nearcnt[p] == 0) nearcnt[p] = nf + pos++;
    __syncthreads();  // (an F list's rank may be 0: written only after every range is done)
    if (threadIdx.x < nf) {
        const unsigned long long mine = s_fkey[threadIdx.x];
        int rank = 0;
        for (int j = 0; j < nf; ++j) rank += s_fkey[j] < mine ? 1 : 0;
        nearcnt[static_cast<int32_t>(mine & 0xFFFFFFFFu)] = rank;
    }
    __syncthreads();
    for (int64_t p = pa; p < pe; ++p) {
        if (maxlen[p] > 0) {
            WorkItem it;
            it.p = static_cast<int32_t>(p);
            it.ext = maxlen[p];
            int e = 0;
            const float m = __int_as_float(maxd1[p]);
            if (m > 0.f) frexpf(m, &e);
            it.sA = m > 0.f ? ldexpf(1.0f, -e) : 1.0f;
            it.sB = sB[p];
            it.radius = radii[p];
            const float c = it.sA / it.sB;  // exact: both powers of two
            it.aug = (c >= 6.103515625e-05f && c <= 32768.0f) ? -c : 0.0f;
            it.poff = static_cast<int32_t>(poff[p]);
            it.csr = static_cast<int32_t>(offsets[p]);
            work[w0 + nearcnt[p]] = it;
        }
    }
    __syncthreads();
    for (int it0 = way * kSegBatch; it0 < cnt; it0 += kFillWays * kSegBatch) {
        uint32_t pb[kSegBatch], lb[kSegBatch];
        load8_u32(reinterpret_cast<const uint32_t *>(seg_list), s0 + it0, cnt - it0, pb, 0u);
        load8_u32(reinterpret_cast<const uint32_t *>(seg_len), s0 + it0, cnt - it0, lb, 0u);
#pragma unroll
        for (int j = 0; j < kSegBatch; ++j)
            if (it0 + j < cnt) cut[(w0 + nearcnt[pb[j]]) * kRows + row] = static_cast<int32_t>(lb[j]);
    }
    if (w0 > wbase) {
        __syncthreads();
        if (threadIdx.x == 0) {
            WorkItem it = work[w0];
            it.csr = -1;  // max-only marker
            work[wbase] = it;
        }
        if (way == 0) cut[wbase * kRows + row] = cut[w0 * kRows + row];
    }
    // LPT: heavier tiles first
    if (threadIdx.x == 0) {
        // 16-bit LPT key: the work as a 5-bit exponent and 11-bit mantissa (monotonic, ~0.05%
        // resolution), so the tile sort needs 16 key bits (two radix passes instead of four)
        const unsigned long long wk = s_work;
        unsigned key = 0;
        if (wk > 0) {
            const int e = min(63 - __clzll(static_cast<long long>(wk)), 31);
            const unsigned m = static_cast<unsigned>(e >= 11 ? (wk >> (e - 11)) : (wk << (11 - e))) & 0x7FFu;
            key = (static_cast<unsigned>(e) << 11) | m;
        }
        tile_key[blockIdx.x] = 0xFFFFull - key;
    }
}

// k > 1: heavy tiles (a few queries whose k-th nearest representative lies in another region
// scan almost every list) are split over several CTAs: the tile's work items in up to
// `maxsplit` contiguous ranges, each a virtual tile with its own candidate slots (split index),
// merged by the re-rank.  A tile is split when its work exceeds half an SM's share; the work
// comes back from the LPT key (16-bit exponent/mantissa code of tile_fill_kernel).
__device__ __forceinline__ double lpt_work(uint64_t tkey) {
    const unsigned key = 0xFFFFu - static_cast<unsigned>(tkey);
    if (key == 0) return 0.0;
    return ldexp(static_cast<double>(0x800u | (key & 0x7FFu)), static_cast<int>(key >> 11) - 11);
}

__global__ void __launch_bounds__(1024) split_plan_kernel(const int32_t *__restrict__ tile_order,
                                                          const uint64_t *__restrict__ tkey_sorted, int ntiles,
                                                          const int64_t *__restrict__ work_off,
                                                          const int64_t *__restrict__ nwork, int maxsplit, int nsm,
                                                          int4 *__restrict__ vt, int32_t *__restrict__ nvt) {
    typedef cub::BlockReduce<double, 1024> Red;
    typedef cub::BlockScan<int, 1024> Scan;
    __shared__ typename Red::TempStorage red_tmp;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ double s_total;
    __shared__ int s_base;
    double part = 0.0;
    for (int i = threadIdx.x; i < ntiles; i += blockDim.x) part += lpt_work(tkey_sorted[i]);
    const double tot = Red(red_tmp).Sum(part);
    if (threadIdx.x == 0) {
        s_total = tot;
        s_base = 0;
    }
    __syncthreads();
    const double half_share = s_total / (2.0 * nsm);
    for (int i0 = 0; i0 < ntiles; i0 += blockDim.x) {
        const int i = i0 + threadIdx.x;
        int S = 0, tile = 0;
        int64_t wo = 0, nw = 0;
        if (i < ntiles) {
            tile = tile_order[i];
            wo = work_off[tile];
            nw = nwork[tile];
            const double W = lpt_work(tkey_sorted[i]);
            S = 1;
            if (half_share > 0.0 && W > half_share) S = min(maxsplit, static_cast<int>(W / half_share) + 1);
            if (S > nw) S = nw > 1 ? static_cast<int>(nw) : 1;
        }
        int pos, total;
        Scan(scan_tmp).ExclusiveSum(S, pos, total);
        const int base = s_base;
        for (int sp = 0; sp < S; ++sp)
            vt[base + pos + sp] = make_int4(tile, static_cast<int>(wo + nw * sp / S), static_cast<int>(wo + nw * (sp + 1) / S), sp);
        __syncthreads();
        if (threadIdx.x == 0) s_base += total;
        __syncthreads();
    }
    if (threadIdx.x == 0) *nvt = s_base;
}

// ---- the stage-2 kernel -----------------------------------------------------------------
template <int KT, int NP>
__global__ void __launch_bounds__(kThreads, 1) stage2_tc_kernel(const S2Params P) {
    using Cfg = S2Cfg<NP>;
    constexpr int kN = Cfg::kN, kStages = Cfg::kStages, kCols = Cfg::kCols, kKd = Cfg::kKd, kAcc = Cfg::kAcc;
    constexpr int kStageBytes = Cfg::kStageBytes, kABytes = Cfg::kABytes;
    constexpr float kAccErrNP = kAccErr * NP;
    if (static_cast<int64_t>(*P.work_total) > P.cap_work) return;  // work arrays incomplete (see tile_fill_kernel)
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024 - (sm100::smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t *sB = smem;                                   // kStages x (plane 0 | plane 1)
    uint8_t *sA = sB + kStages * kStageBytes;             // 2 x (plane 0 | plane 1)
    float *gbuf = reinterpret_cast<float *>(sA + 2 * kABytes);  // 8 epilogue warps x 128 (fallback column)
    float *s_dq = gbuf + kEpiWarps * kCols;  // [4 list slots][kParts][128] partial |q - r_p|^2
    float *s_da = s_dq + 4 * kParts * kRows;  // [4 list slots][kParts][128] partial |a - f16(a)|^2 (scaled)
    float *sQ = s_da + 4 * kParts * kRows;  // NP = 1: [128][kQStride] the tile's query rows
    uint8_t *lring = reinterpret_cast<uint8_t *>(sQ + Cfg::kQSmemFloats);  // [kLSlots] per-list data
    uint64_t *bars = reinterpret_cast<uint64_t *>(lring + kLSlots * Cfg::kLSlotBytes);
    uint64_t *full = bars, *empty = bars + kStages, *tfull = bars + 2 * kStages, *tempty = tfull + kAcc;
    uint64_t *afull = tempty + kAcc, *aempty = afull + 2, *tile_full = aempty + 2, *tile_empty = tile_full + 2;
    uint64_t *lfull = tile_empty + 2, *lempty = lfull + kLSlots;
    uint32_t *s_tmem = reinterpret_cast<uint32_t *>(lempty + kLSlots);
    // list data of ring position li: its work item and representative row (+ dbmax at [64 NP])
    auto lslot_wi = [&](uint32_t li) -> const WorkItem & {
        return *reinterpret_cast<const WorkItem *>(lring + (li % kLSlots) * Cfg::kLSlotBytes);
    };
    auto lslot_rep = [&](uint32_t li) {
        return reinterpret_cast<const float *>(lring + (li % kLSlots) * Cfg::kLSlotBytes + 32);
    };
    auto lslot_cut = [&](uint32_t li) {  // the list's per-row cutoffs (work item's cut row)
        return reinterpret_cast<const int32_t *>(lring + (li % kLSlots) * Cfg::kLSlotBytes + 32 + Cfg::kRepStride * 4);
    };
    int *s_tiles = reinterpret_cast<int *>(s_tmem + 1);  // 2-slot ring of tile ids
    // work items [w0, w1) of scheduled entry t (a virtual tile when heavy tiles are split) and
    // its split index (candidate slots split * kParts + part)
    auto work_range = [&](int t, int64_t &w0, int64_t &w1) -> int {
        if (P.vt) {
            const int4 e = P.vt[t];
            w0 = e.y;
            w1 = e.z;
            return e.w;
        }
        w0 = P.work_off[t];
        w1 = w0 + P.nwork[t];
        return 0;
    };

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    S2_TIME(unsigned long long tw[12] = {});
    S2_TIME(const unsigned long long t_start = clock64());
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            sm100::mbar_init(&full[s], 1);
            sm100::mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < kAcc; ++b) {
            sm100::mbar_init(&tfull[b], 1);
            sm100::mbar_init(&tempty[b], kEpiWarps);
        }
        for (int b = 0; b < 2; ++b) {
            sm100::mbar_init(&afull[b], kEpiWarps);
            sm100::mbar_init(&aempty[b], 1);
            sm100::mbar_init(&tile_full[b], 1);
            sm100::mbar_init(&tile_empty[b], 1 + kEpiWarps);  // MMA lane + epilogue warps
        }
        for (int l = 0; l < kLSlots; ++l) {
            sm100::mbar_init(&lfull[l], 1);
            sm100::mbar_init(&lempty[l], kEpiWarps);
        }
        sm100::fence_barrier_init();
    }
    if (warp == 1) sm100::tmem_alloc<Cfg::kTmemCols>(s_tmem);
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    const uint32_t tmem = *s_tmem;

    if (warp == 0) {
        // ===== scheduler + producer =====
        sm100::setmaxnreg_dec<kRegsCtl>();
        if (lane == 0) {
            uint32_t bi = 0, li = 0;
            // list data of work item w into the next ring slot (the epilogue prepares list w + 1's
            // A operand while list w's chunks run, so w + 1's data is issued before w's chunks)
            auto issue_list = [&](int64_t w) {
                const uint32_t sl = li % kLSlots;
                sm100::mbar_wait(&lempty[sl], ((li / kLSlots) & 1) ^ 1);
                uint8_t *dst = lring + sl * Cfg::kLSlotBytes;
                const int32_t p = P.work[w].p;
                sm100::mbar_arrive_expect_tx(&lfull[sl], 32 + Cfg::kRepStride * 4 + (P.cut ? kRows * 4 : 0));
                sm100::bulk_g2s(dst, P.work + w, 32, &lfull[sl]);
                sm100::bulk_g2s(dst + 32, P.reps64 + static_cast<int64_t>(p) * Cfg::kRepStride, Cfg::kRepStride * 4,
                                &lfull[sl]);
                if (P.cut)
                    sm100::bulk_g2s(dst + 32 + Cfg::kRepStride * 4, P.cut + w * kRows, kRows * 4, &lfull[sl]);
                ++li;
            };
            for (uint32_t it = 0;; ++it) {
                const uint32_t slot = it & 1;
                sm100::mbar_wait(&tile_empty[slot], ((it >> 1) & 1) ^ 1);
                const int t = atomicAdd(P.tile_counter, 1);
                const int tile = P.vt ? (t < *P.nvt ? t : -1) : (t < P.ntiles ? P.tile_order[t] : -1);
                s_tiles[slot] = tile;
                sm100::mbar_arrive(&tile_full[slot]);
                if (tile < 0) break;
                int64_t wt0, wt1;
                work_range(tile, wt0, wt1);
                if (wt0 < wt1) issue_list(wt0);
                for (int64_t w = wt0, w1 = wt1; w < w1; ++w) {
                    if (w + 1 < w1) issue_list(w + 1);
                    const WorkItem wi = P.work[w];
                    for (int off = 0; off < wi.ext; off += kN) {
                        const int n = min(kN, roundup16(wi.ext - off));
                        const uint32_t s = bi % kStages;
                        S2_WAIT(&empty[s], ((bi / kStages) & 1) ^ 1, 0);
                        uint8_t *dst = sB + s * kStageBytes;
                        const uint32_t b0 = static_cast<uint32_t>(n) * kP0;
                        const uint32_t b1 = P.plane1 ? static_cast<uint32_t>(n) * kP1 : 0u;
#ifdef RBC_S2_NOLOAD
                        if (P.cut) {  // diagnostic: no B traffic in the search (stale operands, results invalid)
                            sm100::mbar_arrive(&full[s]);
                            ++bi;
                            continue;
                        }
#endif
                        sm100::mbar_arrive_expect_tx(&full[s], NP * b0 + b1);
#pragma unroll
                        for (int j = 0; j < NP; ++j)
                            sm100::bulk_g2s(dst + j * kN * kP0,
                                            P.xh0 + j * P.plane_bytes + (static_cast<int64_t>(wi.poff) + off) * kP0, b0,
                                            &full[s]);
                        if (b1)
                            sm100::bulk_g2s(dst + NP * kN * kP0, P.xh1 + (static_cast<int64_t>(wi.poff) + off) * kP1, b1,
                                            &full[s]);
                        ++bi;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer =====
        sm100::setmaxnreg_dec<kRegsCtl>();
        if (lane == 0) {
            uint32_t bi = 0, ti = 0, ai = 0, li = 0;
            for (uint32_t it = 0;; ++it) {
                const uint32_t slot = it & 1;
                sm100::mbar_wait(&tile_full[slot], (it >> 1) & 1);
                const int tile = s_tiles[slot];
                sm100::mbar_arrive(&tile_empty[slot]);
                if (tile < 0) break;
                int64_t w, w1;
                work_range(tile, w, w1);
                for (; w < w1; ++w, ++li) {
                    sm100::mbar_wait(&lfull[li % kLSlots], (li / kLSlots) & 1);
                    const int ext = lslot_wi(li).ext;
                    const uint32_t a = ai & 1;
                    S2_WAIT(&afull[a], (ai >> 1) & 1, 1);
                    sm100::tc_fence_after();
                    const uint32_t a0 = sm100::smem_u32(sA + a * kABytes);
                    for (int off = 0; off < ext; off += kN) {
                        const int n = min(kN, roundup16(ext - off));
                        const uint32_t s = bi % kStages, tb = ti % kAcc;
                        S2_WAIT(&full[s], (bi / kStages) & 1, 2);
                        S2_WAIT(&tempty[tb], ((ti / kAcc) & 1) ^ 1, 3);
                        sm100::tc_fence_after();
                        const uint32_t idesc = sm100::idesc_f16_f32(kRows, static_cast<uint32_t>(n));
                        const uint32_t b0 = sm100::smem_u32(sB + s * kStageBytes);
                        const uint32_t d_tmem = tmem + tb * kN;
#pragma unroll
                        for (int j = 0; j < NP; ++j)
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk)
                                sm100::umma_f16(d_tmem, sm100::umma_desc_sw128(a0 + j * kRows * kP0 + kk * 32),
                                                sm100::umma_desc_sw128(b0 + j * kN * kP0 + kk * 32), idesc,
                                                (j | kk) > 0);
                        if (P.plane1)
                            sm100::umma_f16(d_tmem, sm100::umma_desc_sw32(a0 + NP * kRows * kP0),
                                            sm100::umma_desc_sw32(b0 + NP * kN * kP0), idesc, 1);
                        sm100::umma_commit(&empty[s]);
                        sm100::umma_commit(&tfull[tb]);
                        ++bi;
                        ++ti;
                    }
                    sm100::umma_commit(&aempty[a]);
                    ++ai;
                }
            }
        }
    } else if (warp < kEpiWarp0) {
        sm100::setmaxnreg_dec<kRegsCtl>();  // idle warps of warp group 0
    } else {
        // ===== epilogue warps (kParts per TMEM lane quadrant): A prep + filter + candidate buffer =====
        sm100::setmaxnreg_inc<kRegsEpi>();
        // warp (quad, part): rows quad*32 .. +31, columns [part*kCols, +kCols) of every 256-column
        // chunk (two 32-column halves), K range [part*kKd, +kKd) of the A operand.
        const int quad = warp & 3;
        const int part = (warp - kEpiWarp0) >> 2;
        const int row = quad * 32 + lane;
        float *g = gbuf + (warp - kEpiWarp0) * kCols;
        uint32_t ti = 0, ai = 0, li0 = 0;  // li0: ring position of the tile's first list
        for (uint32_t it = 0;; ++it) {
            const uint32_t slot = it & 1;
            sm100::mbar_wait(&tile_full[slot], (it >> 1) & 1);
            const int tile = s_tiles[slot];
            __syncwarp();
            if (lane == 0) sm100::mbar_arrive(&tile_empty[slot]);
            if (tile < 0) break;
            int64_t w0, w1;
            const int split = work_range(tile, w0, w1);
            const int64_t slot_q = static_cast<int64_t>(P.vt ? P.vt[tile].x : tile) * kRows + row;
            const int32_t qi = slot_q < P.nq ? P.order[slot_q] : -1;
            const bool live = qi >= 0;
            // this thread's quarter of the query row (rows padded to 64 floats with zeros)
            // (NP = 2: 64 floats per thread would not fit beside the epilogue's registers;
            // prep_a then re-reads the row from L1)
            const float4 *qsrc =
                reinterpret_cast<const float4 *>(P.q64 + static_cast<int64_t>(live ? qi : 0) * (64 * NP) + part * kKd);
            // NP = 1: this thread's part of its query row into shared memory (only this thread
            // reads it back, in prep_a; the previous tile's reads by this thread are done)
            float4 *qs4 = reinterpret_cast<float4 *>(sQ + row * Cfg::kQStride + part * kKd);
            if (NP == 1) {
#pragma unroll
                for (int c = 0; c < kKd / 4; ++c) qs4[c] = live ? __ldg(qsrc + c) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            // A operand of list w: this thread's kKd * 2 bytes of row `row` (+ the aug columns, last part)
            auto prep_a = [&](int64_t w) {
                S2_TIME(const unsigned long long tp0 = clock64());
                S2_TIME(++tw[11]);
                const uint32_t lw = li0 + static_cast<uint32_t>(w - w0);
                sm100::mbar_wait(&lfull[lw % kLSlots], (lw / kLSlots) & 1);
                const WorkItem wi = lslot_wi(lw);
                const float4 *rep4 = reinterpret_cast<const float4 *>(lslot_rep(lw) + part * kKd);
                const __half ac = __float2half_rn(wi.aug);
                const uint32_t aug = static_cast<uint32_t>(__half_as_ushort(ac)) * 0x00010001u;
                const float sa = wi.sA;
                const uint32_t a = ai & 1;
                // one 16-byte chunk (8 dims) of this thread's K range: f16 residuals, their rounding
                // error, and the chunk's share of |q - r_p|^2
                auto chunk = [&](int c, const float *qq, const float *rr, float &nq2, float &da2) {
                    uint32_t wv[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float v0 = fmaf(qq[2 * e], sa, -(rr[2 * e] * sa));
                        const float v1 = fmaf(qq[2 * e + 1], sa, -(rr[2 * e + 1] * sa));
                        wv[e] = sm100::pack_f16x2_sat(v0, v1);
                        __half2 h;
                        *reinterpret_cast<uint32_t *>(&h) = wv[e];
                        const float2 hf2 = __half22float2(h);
                        const float e0 = v0 - hf2.x, e1 = v1 - hf2.y;
                        da2 = fmaf(e0, e0, fmaf(e1, e1, da2));
                    }
                    // global 16-byte chunk index -> (plane, chunk in the 128-byte row)
                    const int g = part * (kKd / 8) + c, pl = g >> 3, cc = g & 7;
                    if (!P.plane1 && g == 8 * NP - 1) wv[3] = aug;
                    uint8_t *dst = sA + a * kABytes + pl * kRows * kP0 + row * kP0;
                    *reinterpret_cast<uint4 *>(dst + ((cc ^ (row & 7)) << 4)) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
                };
                float da2 = 0.f;  // |a - f16(a)|^2 of this part (scaled units)
                if constexpr (NP == 1) {
                    float4 rr4[kKd / 4];
                    float qv[kKd];
#pragma unroll
                    for (int c = 0; c < kKd / 4; ++c) {
                        rr4[c] = rep4[c];
                        const float4 t = qs4[c];
                        qv[4 * c] = t.x;
                        qv[4 * c + 1] = t.y;
                        qv[4 * c + 2] = t.z;
                        qv[4 * c + 3] = t.w;
                    }
                    // this part's share of |q - r_p|^2 (fp32; with the other part's, the A2 term of
                    // the error bound -- same (d + 2) 2^-24 relative error budget as kD1 / kUq)
                    {
                        float n0 = 0.f, n1 = 0.f;
#pragma unroll
                        for (int c = 0; c < kKd / 4; ++c) {
                            const float t0 = qv[4 * c] - rr4[c].x, t1 = qv[4 * c + 1] - rr4[c].y;
                            const float t2 = qv[4 * c + 2] - rr4[c].z, t3 = qv[4 * c + 3] - rr4[c].w;
                            n0 = fmaf(t0, t0, fmaf(t1, t1, n0));
                            n1 = fmaf(t2, t2, fmaf(t3, t3, n1));
                        }
                        s_dq[(static_cast<int>(w) & 3) * (kParts * kRows) + part * kRows + row] = n0 + n1;
                    }
                    S2_WAIT(&aempty[a], ((ai >> 1) & 1) ^ 1, 4);
#pragma unroll
                    for (int c = 0; c < kKd / 8; ++c) {
                        const float rr[8] = {rr4[2 * c].x, rr4[2 * c].y, rr4[2 * c].z, rr4[2 * c].w,
                                             rr4[2 * c + 1].x, rr4[2 * c + 1].y, rr4[2 * c + 1].z, rr4[2 * c + 1].w};
                        float nd = 0.f;
                        chunk(c, qv + 8 * c, rr, nd, da2);
                    }
                } else {
                    // NP = 2: 64 dims per thread, streamed 8 at a time (query and rep rows from L1)
                    S2_WAIT(&aempty[a], ((ai >> 1) & 1) ^ 1, 4);
                    float n0 = 0.f, n1 = 0.f;
#pragma unroll 2
                    for (int c = 0; c < kKd / 8; ++c) {
                        const float4 r0 = rep4[2 * c], r1 = rep4[2 * c + 1];
                        const float4 q0 = live ? __ldg(qsrc + 2 * c) : make_float4(0.f, 0.f, 0.f, 0.f);
                        const float4 q1 = live ? __ldg(qsrc + 2 * c + 1) : make_float4(0.f, 0.f, 0.f, 0.f);
                        const float rr[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
                        const float qq[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float t0 = qq[2 * e] - rr[2 * e], t1 = qq[2 * e + 1] - rr[2 * e + 1];
                            n0 = fmaf(t0, t0, n0);
                            n1 = fmaf(t1, t1, n1);
                        }
                        float nd = 0.f;
                        chunk(c, qq, rr, nd, da2);
                    }
                    s_dq[(static_cast<int>(w) & 3) * (kParts * kRows) + part * kRows + row] = n0 + n1;
                }
                s_da[(static_cast<int>(w) & 3) * (kParts * kRows) + part * kRows + row] = da2;
                if (P.plane1 && part == kParts - 1) {
                    uint8_t *d1p = sA + a * kABytes + NP * kRows * kP0 + row * kP1;
                    const int sw = (row >> 2) & 1;
                    *reinterpret_cast<uint4 *>(d1p + ((0 ^ sw) << 4)) = make_uint4(aug, 0, 0, 0);
                    *reinterpret_cast<uint4 *>(d1p + ((1 ^ sw) << 4)) = make_uint4(0, 0, 0, 0);
                }
                sm100::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) sm100::mbar_arrive(&afull[a]);
                ++ai;
                S2_TIME(tw[8] += clock64() - tp0);
            };
            if (w0 < w1) prep_a(w0);

            float ubk[KT];
#pragma unroll
            for (int j = 0; j < KT; ++j) ubk[j] = __int_as_float(0x7f800000);
            const float gk = live ? P.gamma[qi] : 0.f;
            const float u_init = gk * gk * kUp * kUp;
            float U = u_init;  // running upper bound of the k-th smallest candidate d^2
            int count = 0;     // buffered 8-column groups
            bool overflow = false;
            // k = 1: the newest qualifying group (values, their max, (lb0, 2/scale, valid), position)
            float hv[9];
            float4 hm = make_float4(0.f, 0.f, 0.f, 0.f);
            int32_t hpos = 0;
            bool held = false;
            const int64_t slot_id = static_cast<int64_t>(live ? qi : 0) * P.nslot + split * kParts + part;
            float4 *clb = reinterpret_cast<float4 *>(P.cand_lb) + slot_id * P.cap * 3;
            int32_t *cpos = P.cand_pos + slot_id * P.cap;
            for (int64_t w = w0; w < w1; ++w) {
                if (w + 1 < w1) prep_a(w + 1);  // next list's A while this list's MMAs run
                const uint32_t lw = li0 + static_cast<uint32_t>(w - w0);  // (waited for by prep_a(w))
                const WorkItem wi = lslot_wi(lw);
                const int cutv = live ? (P.cut ? lslot_cut(lw)[row] : wi.ext) : 0;
                // both column parts of this lane quadrant have prepared lists w and w + 1: the
                // row's |q - r_p|^2 is the sum of their two halves (slot w & 3; a part runs at
                // most one list ahead of its partner, so slots are never overwritten early)
                asm volatile("bar.sync %0, %1;" ::"r"(1 + quad), "r"(32 * kParts) : "memory");
                float A2q = 0.f, DA2 = 0.f;
#pragma unroll
                for (int h = 0; h < kParts; ++h) {
                    A2q += s_dq[(static_cast<int>(w) & 3) * (kParts * kRows) + h * kRows + row];
                    DA2 += s_da[(static_cast<int>(w) & 3) * (kParts * kRows) + h * kRows + row];
                }
                const float dq = sqrtf(A2q);
                const bool noaug = wi.aug == 0.0f;  // warp-uniform (per work item)
                const float sa = wi.sA;
                const float scale = sa * wi.sB, inv2s = 2.0f / scale;
                float A2 = 0.f, E = 0.f;
                if (cutv > 0) {
                    // A2 = |q - r_p|^2 in fp32 with relative error <= (d + 2) 2^-24 -- covered by
                    // kD1 (on A2) and kUq (on |a| = sqrt(A2))
                    const float na = dq * kUq, rb = wi.radius * kUp;
                    A2 = A2q;
                    // f16 rounding of the operands from the actual rounding errors: |dot(f16 a,
                    // f16 b) - a.b| <= |da||b| + |a||db| + |da||db| (Cauchy-Schwarz), with |da|
                    // this row's A error and |db| the list's largest B error (unscaled; +2^-23
                    // relative for the fp32 residual rounding before the f16 conversion), x2 for
                    // d^2 and x2 safety as in kC1; fp32 accumulation keeps its kC1 share
                    const float da = sqrtf(DA2) * (1.0f + 1.0f / 1024.0f) / sa + dq * (1.0f / 8388608.0f);
                    const float db = lslot_rep(lw)[64 * NP] * (1.0f + 1.0f / 1024.0f) / wi.sB + rb * (1.0f / 8388608.0f);
                    E = 4.0f * (da * rb + na * db + da * db) + kAccErrNP * na * rb + kC2 * (A2 + rb * rb) + kD1 * A2 +
                        kC4 * rb * (2.0f / sa) + 1e-30f;
                }
                const float lb0 = A2 - E;  // lb(V) = lb0 - V * inv2s
                // V >= T  <=>  lb = A2 - E - 2 V / scale <= U * kTie   (loosened by 2^-18 relative)
                auto threshold = [&]() {
                    const float t = 0.5f * scale * (A2 - E - U * kTie);
                    return t - fabsf(t) * (1.0f / 262144.0f) - 1e-30f;
                };
                const bool maxonly = wi.csr < 0;  // warm-up copy: bound only, no candidates
                float T = (cutv > 0 && !maxonly) ? threshold() : __int_as_float(0x7f800000);
                float vbest = -__int_as_float(0x7f800000);
                // compact the buffer (once per 32-column half) when it could fill up
                auto compact = [&]() {
                    const float ut = U * kTie;
                    int c2 = 0;
                    // kCB groups loaded before any is written back: the loads are independent (in
                    // flight together) and every write-back slot c2 <= e precedes the batch's
                    // unread entries, so nothing is overwritten before it is read
                    constexpr int kCB = KT == 1 ? 1 : 4;  // (k = 1 rarely compacts: no registers for it)
                    for (int e0 = 0; e0 < count; e0 += kCB) {
                        float4 a[kCB], b[kCB], c[kCB];
                        int32_t ps[kCB];
#pragma unroll
                        for (int j = 0; j < kCB; ++j) {
                            const int e = e0 + j < count ? e0 + j : e0;
                            a[j] = clb[3 * e];
                            b[j] = clb[3 * e + 1];
                            c[j] = clb[3 * e + 2];
                            ps[j] = cpos[e];
                        }
#pragma unroll
                        for (int j = 0; j < kCB; ++j) {
                            const float vmax = fmaxf(fmaxf(fmaxf(a[j].x, a[j].y), fmaxf(a[j].z, a[j].w)),
                                                     fmaxf(fmaxf(b[j].x, b[j].y), fmaxf(b[j].z, b[j].w)));
                            // the group's smallest lower bound (all 8 columns)
                            if (e0 + j < count && fmaf(-vmax, c[j].y, c[j].x) <= ut) {
                                clb[3 * c2] = a[j];
                                clb[3 * c2 + 1] = b[j];
                                clb[3 * c2 + 2] = c[j];
                                cpos[c2] = ps[j];
                                ++c2;
                            }
                        }
                    }
                    count = c2;
                };
                // buffer a whole 8-column group -- the raw accumulator values plus (lb0, 2/scale,
                // valid columns): lb = lb0 - V * 2/scale, computed by the re-rank -- and tighten
                // the bound with the group's best element; the exact re-rank filters
                auto push8 = [&](const float *v, float m, int col0, int lim, bool block_valid) {
                    if (KT == 1 && kHold) {
                        // k = 1: the newest qualifying group is held in registers; the one it
                        // replaces is stored only if it can still hold the nearest candidate
                        // (its smallest lower bound is within the current bound) -- usually the
                        // new group has just improved on it
                        if (held && fmaf(-hv[8], hm.y, hm.x) <= U * kTie) {
                            if (count < P.cap) {
                                clb[3 * count] = make_float4(hv[0], hv[1], hv[2], hv[3]);
                                clb[3 * count + 1] = make_float4(hv[4], hv[5], hv[6], hv[7]);
                                clb[3 * count + 2] = hm;
                                cpos[count] = hpos;
                                ++count;
                            } else {
                                overflow = true;
                            }
                        }
#pragma unroll
                        for (int j = 0; j < 8; ++j) hv[j] = v[j];
                        hv[8] = m;
                        hm = make_float4(lb0, inv2s, __int_as_float(min(8, lim - col0)), 0.f);
                        hpos = wi.csr + col0;
                        held = true;
                    } else if (count < P.cap) {
                        clb[3 * count] = make_float4(v[0], v[1], v[2], v[3]);
                        clb[3 * count + 1] = make_float4(v[4], v[5], v[6], v[7]);
                        clb[3 * count + 2] = make_float4(lb0, inv2s, __int_as_float(min(8, lim - col0)), 0.f);
                        cpos[count] = wi.csr + col0;
                        ++count;
                    } else {
                        overflow = true;
                    }
                    // the group's best is a valid element: its ub bounds the k-th best (k = 1 and a
                    // fully valid block: the block maximum already did).  (Every element's ub into
                    // the k-best set instead, for k > 1, measured no fewer buffered groups: the
                    // pushes follow the k-record statistics of the scan order, ~k ln(N/k).)
                    if (col0 + 8 <= lim && (KT > 1 || !block_valid)) {
                        const float ub = fmaf(-m, inv2s, lb0) + 2.0f * E;
                        if (KT == 1) {
                            U = fminf(U, ub);
                        } else {
                            float x = ub;
#pragma unroll
                            for (int t = 0; t < KT; ++t) {
                                const float lo = fminf(ubk[t], x), hi = fmaxf(ubk[t], x);
                                ubk[t] = lo;
                                x = hi;
                            }
                            float kth = ubk[KT - 1];
                            if (KT != 10 && P.k != KT) {  // (KT = 10 serves k = 10 only)
#pragma unroll
                                for (int t = 0; t < KT; ++t)
                                    if (t == P.k - 1) kth = ubk[t];
                            }
                            U = fminf(u_init, kth);
                        }
                        T = threshold();
                    }
                };
                for (int off = 0; off < wi.ext; off += kN) {
                    const int n = min(kN, roundup16(wi.ext - off));
                    const int hb = part * kCols;  // this warp's first column in the chunk
                    if (noaug) {
                        // rare: per-column norm term subtracted here instead of in the MMA
                        const float *src = P.gcol + wi.poff + off + hb;
                        for (int c = lane; c < kCols; c += 32) g[c] = hb + c < n ? src[c] : 0.f;
                    }
                    const uint32_t tb = ti % kAcc;
                    S2_WAIT(&tfull[tb], (ti / kAcc) & 1, 5);
                    sm100::tc_fence_after();
                    __syncwarp();
                    // valid columns of this row, relative to this warp's part of the chunk
                    const int lim = min(min(cutv - off, n) - hb, kCols);
#ifdef RBC_S2_NOEPI
                    // diagnostic: pipeline without epilogue work in the search (results invalid; the
                    // build's brute force keeps its epilogue so the index is still right)
                    const int wlim = P.cut ? 0 : __reduce_max_sync(0xffffffffu, max(lim, 0));
#else
                    const int wlim = __reduce_max_sync(0xffffffffu, max(lim, 0));
#endif
                    const uint32_t tbase = tmem + tb * kN + hb + (static_cast<uint32_t>(quad * 32) << 16);
                    // one 32-column block of this warp's columns: max tree against the running
                    // bound, candidate groups buffered on the slow path
                    auto block = [&](uint32_t (&ra)[32], const int c0) {
#if defined(RBC_S2_LEVEL) && RBC_S2_LEVEL == 1
                        if (P.cut) {  // diagnostic: TMEM loads only (search only)
                            uint32_t x = 0;
#pragma unroll
                            for (int j = 0; j < 32; ++j) x ^= ra[j];
                            if (x == 0x12345u) count += 1;
                            return;
                        }
#endif
                        float va[32];
#pragma unroll
                        for (int j = 0; j < 32; ++j) va[j] = __uint_as_float(ra[j]);
                        if (noaug) {
#pragma unroll
                            for (int j = 0; j < 32; ++j) va[j] = fmaf(-sa, g[c0 + j], va[j]);
                        }
                        float m8[4];
#pragma unroll
                        for (int s = 0; s < 4; ++s) m8[s] = max8(va + 8 * s);
                        const float ma = sm100::fmax3(m8[0], m8[1], fmaxf(m8[2], m8[3]));
                        if (KT == 1) {
                            // k = 1: a fully valid half's best element bounds the nearest candidate
                            if (c0 + 32 <= lim && ma > vbest) {
                                vbest = ma;
                                const float ub = fmaf(-ma, inv2s, lb0) + 2.0f * E;
                                if (ub < U) {
                                    U = ub;
                                    if (!maxonly) T = threshold();
                                }
                            }
                        }
#if defined(RBC_S2_LEVEL) && RBC_S2_LEVEL == 2
                        if (P.cut) {  // diagnostic: loads + reductions, no candidates (search only)
                            if (ma == 1234.5f) count += 1;
                            return;
                        }
#endif
                        if (ma >= T) {
                            if (count + 4 > P.cap && !overflow) compact();
                            const int base = off + hb + c0, llim = off + hb + lim;
#pragma unroll
                            for (int s = 0; s < 4; ++s)
                                if (m8[s] >= T) push8(va + 8 * s, m8[s], base + 8 * s, llim, c0 + 32 <= lim);
                        }
                    };
#if defined(RBC_S2_X64)
                    // diagnostic variant: one 64-column TMEM round trip per two blocks
                    for (int c0 = 0; c0 < wlim; c0 += 64) {
                        uint32_t r64[64];
                        sm100::tmem_ld64_wait(tbase + c0, r64);
                        block(*reinterpret_cast<uint32_t(*)[32]>(r64), c0);
                        if (c0 + 32 < wlim) block(*reinterpret_cast<uint32_t(*)[32]>(r64 + 32), c0 + 32);
                    }
#elif defined(RBC_S2_PIPE)
                    // diagnostic variant: block b + 1's TMEM load in flight while block b is reduced
                    // (measured slower: cfg2 stage 2 0.51 -> 0.70 ms)
                    uint32_t ra[32], rb[32];
                    if (wlim > 0) {
                        sm100::tmem_ld32_async(tbase, ra);
                        sm100::tmem_wait_ld(ra);
                    }
#pragma unroll 1
                    for (int c0 = 0; c0 < wlim; c0 += 64) {
                        const bool n1 = c0 + 32 < wlim, n2 = c0 + 64 < wlim;
                        if (n1) sm100::tmem_ld32_async(tbase + c0 + 32, rb);
                        block(ra, c0);
                        __syncwarp();
                        if (!n1) break;
                        sm100::tmem_wait_ld(rb);
                        if (n2) sm100::tmem_ld32_async(tbase + c0 + 64, ra);
                        block(rb, c0 + 32);
                        __syncwarp();
                        if (n2) sm100::tmem_wait_ld(ra);
                    }
#else
                    for (int c0 = 0; c0 < wlim; c0 += 32) {
                        uint32_t ra[32];
                        sm100::tmem_ld32_async(tbase + c0, ra);
                        sm100::tmem_wait_ld(ra);
                        block(ra, c0);
                    }
#endif
                    sm100::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) sm100::mbar_arrive(&tempty[tb]);
                    ++ti;
                }
                // list w's ring slot is free once every epilogue warp is past it
                __syncwarp();
                if (lane == 0) sm100::mbar_arrive(&lempty[lw % kLSlots]);
            }
            li0 += static_cast<uint32_t>(w1 - w0);
            // the held group joins the buffer (k = 1)
            if (KT == 1 && kHold && held && !overflow) {
                if (count < P.cap) {
                    clb[3 * count] = make_float4(hv[0], hv[1], hv[2], hv[3]);
                    clb[3 * count + 1] = make_float4(hv[4], hv[5], hv[6], hv[7]);
                    clb[3 * count + 2] = hm;
                    cpos[count] = hpos;
                    ++count;
                } else {
                    overflow = true;
                }
            }
            // hand the buffered candidates to the exact re-rank kernel
            if (live) {
                P.cand_count[slot_id] = overflow ? -1 : count;
                P.cand_ufin[slot_id] = U * kTie;
                if (overflow) P.overflow_list[atomicAdd(P.overflow_count, 1)] = qi;
            }
        }
    }
#ifdef RBC_S2_TIMING
    if (P.timing && lane == 0 && (warp <= 1 || warp == kEpiWarp0)) {
        // warp 0: producer, warp 1: MMA, warp 2: one epilogue warp (wait slots 0..5, 6 = role busy-until-exit)
        tw[6] = clock64() - t_start;
        for (int j = 0; j < 12; ++j)
            if (tw[j]) atomicAdd(&P.timing[blockIdx.x * 12 + j], tw[j]);
    }
#endif
    sm100::tc_fence_before();
    __syncthreads();
    if (warp == 1) sm100::tmem_dealloc<Cfg::kTmemCols>(tmem);
}

// Exact re-rank (reference arithmetic) of the buffered candidate groups of both
// column parts: one 8-lane group per query (4 queries per warp), lanes over the
// query's buffered 8-column groups (all groups in flight at once; ~7 per query
// at cfg2), each lane re-ranking its group's elements that can still qualify
// (lb <= final bound, ~1.4 per query); a lane top-k merge emits the keys.
constexpr int kRerankLanes = 8;
constexpr int kRerankThreads = 256;

template <int KT, int DL>
__global__ void __launch_bounds__(kRerankThreads, KT == 1 ? 4 : 0) rerank_kernel(const float4 *__restrict__ cand_lb,
                                                     const int32_t *__restrict__ cand_pos,
                                                     const int32_t *__restrict__ cand_count,
                                                     const float *__restrict__ cand_ufin, int cap, int nslot, int64_t nq,
                                                     const float *__restrict__ q, const float *__restrict__ xp,
                                                     const int32_t *__restrict__ perm, int d, int k,
                                                     uint64_t *__restrict__ out_keys) {
    const int sub = threadIdx.x & (kRerankLanes - 1);
    const int64_t i = (blockIdx.x * static_cast<int64_t>(kRerankThreads) + threadIdx.x) / kRerankLanes;
    if ((blockIdx.x * static_cast<int64_t>(kRerankThreads) + (threadIdx.x & ~31)) / kRerankLanes >= nq) return;
    bool live = i < nq;
    // slots: column parts x splits of a heavy tile (k > 1).  The final bound is the smallest of
    // the slots' bounds: each is at least the k-th best of the union (it bounds the k-th best of
    // its own share).  Split slots that buffered nothing may be unwritten: their bound is skipped.
    constexpr int kSlots = KT == 1 ? kParts : kMaxSlots;  // k = 1 never splits tiles
    const int ns = KT == 1 ? kParts : nslot;
    int cnt[kSlots];
    float ufin = __int_as_float(0x7f800000);
#pragma unroll
    for (int h = 0; h < kSlots; ++h) {
        cnt[h] = (live && h < ns) ? cand_count[static_cast<int64_t>(ns) * i + h] : 0;
        if (cnt[h] < 0) live = false;  // overflowed: recomputed by the exact scan
        if (live && h < ns && (h < kParts || cnt[h] > 0))
            ufin = fminf(ufin, cand_ufin[static_cast<int64_t>(ns) * i + h]);
    }
    int n = 0;
#pragma unroll
    for (int h = 0; h < kSlots; ++h) n += live ? cnt[h] : 0;
    const float *qrow = q + (live ? i : 0) * d;
    uint64_t best[KT];
#pragma unroll
    for (int j = 0; j < KT; ++j) best[j] = kEmptyKey;
    // lanes over the query's buffered groups: the elements that can still qualify
    const int nmax = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(n));
    // group-cooperative exact distances for d <= 8 DL: lane `sub` owns coordinates
    // [sub DL, sub DL + DL) (zero beyond d: exact zero terms do not change the sum)
    const bool fast = d <= kRerankLanes * DL;  // warp-uniform
    const bool vec = fast && (d & 3) == 0 && (reinterpret_cast<uintptr_t>(q) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(xp) & 15) == 0;
    // coordinates of lane `sub`: 16-byte rows -> float4 number sub + 8 t4 (the group's loads
    // of one row are contiguous 128-byte runs); otherwise the run [sub DL, sub DL + DL)
    auto coord = [&](int t) { return vec ? 4 * (sub + kRerankLanes * (t >> 2)) + (t & 3) : sub * DL + t; };
    const bool full = vec && d == kRerankLanes * DL;  // every lane's coordinates inside the row
    float xs[DL];
    if (full) {
#pragma unroll
        for (int t = 0; t < DL; t += 4) {
            const float4 v = live ? __ldg(reinterpret_cast<const float4 *>(qrow) + sub + kRerankLanes * (t >> 2))
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
            xs[t] = v.x;
            xs[t + 1] = v.y;
            xs[t + 2] = v.z;
            xs[t + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int t = 0; t < DL; ++t) xs[t] = (fast && live && coord(t) < d) ? __ldg(qrow + coord(t)) : 0.f;
    }
    // this lane's DL coordinates of point row p
    auto load_row = [&](int32_t p, float (&ys)[DL]) {
        const float *row = xp + static_cast<int64_t>(p) * d;
        if (full) {
            const float4 *r4 = reinterpret_cast<const float4 *>(row) + sub;
#pragma unroll
            for (int t = 0; t < DL; t += 4) {
                const float4 v = __ldg(r4 + kRerankLanes * (t >> 2));
                ys[t] = v.x;
                ys[t + 1] = v.y;
                ys[t + 2] = v.z;
                ys[t + 3] = v.w;
            }
        } else if (vec) {
#pragma unroll
            for (int t = 0; t < DL; t += 4) {
                const float4 v = coord(t) < d ? __ldg(reinterpret_cast<const float4 *>(row + coord(t)))
                                              : make_float4(0.f, 0.f, 0.f, 0.f);
                ys[t] = v.x;
                ys[t + 1] = v.y;
                ys[t + 2] = v.z;
                ys[t + 3] = v.w;
            }
        } else {
#pragma unroll
            for (int t = 0; t < DL; ++t) ys[t] = coord(t) < d ? __ldg(row + coord(t)) : 0.f;
        }
    };
    const int gshift = (threadIdx.x & 31) & ~(kRerankLanes - 1);
    for (int g0 = 0; g0 < nmax; g0 += kRerankLanes) {
        const int g = g0 + sub;
        unsigned pass = 0;
        int32_t pos = 0;
        if (g < n) {
            int h = 0, gg = g;
#pragma unroll
            for (int u = 0; u < kSlots - 1; ++u)
                if (h == u && gg >= cnt[u]) {
                    gg -= cnt[u];
                    h = u + 1;
                }
            const int64_t at = (static_cast<int64_t>(ns) * i + h) * cap + gg;
            const float4 v0 = cand_lb[3 * at], v1 = cand_lb[3 * at + 1], mt = cand_lb[3 * at + 2];
            pos = cand_pos[at];
            const float v[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
            const int valid = __float_as_int(mt.z);
#pragma unroll
            for (int j = 0; j < 8; ++j) pass |= (j < valid && fmaf(-v[j], mt.y, mt.x) <= ufin ? 1u : 0u) << j;
        }
        if (!fast) {  // generic d: each lane re-ranks its own group's elements
            while (pass) {
                const int j = __ffs(pass) - 1;
                pass &= pass - 1;
                const float dist = exact_dist<RBC_L2, 8>(qrow, xp + static_cast<int64_t>(pos + j) * d, d);
                const uint64_t key = pack_key(dist, static_cast<uint32_t>(perm[pos + j]));
                if (key < best[KT - 1]) sorted_insert<KT>(best, key);
            }
            continue;
        }
        // d <= 8 DL: two elements at a time per group (two row loads in flight), the 8 lanes each
        // summing DL of the reference terms of each (identical fp64 terms; only the
        // association differs), then a shuffle tree.  The fp32 result equals the reference's
        // sequential sum unless the tree sum's square root lies within 2^-44 (relative) of an
        // fp32 rounding midpoint -- the two sums differ by at most 2 * 127 * 2^-53 relative --
        // in which case the owner lane recomputes the sequential sum.
        auto finish = [&](double part, int32_t pp) {
            const double r = __dsqrt_rn(part);
            float f = __double2float_rn(r);
            const double mlo = 0.5 * (static_cast<double>(f) + static_cast<double>(nextafterf(f, -INFINITY)));
            const double mhi = 0.5 * (static_cast<double>(f) + static_cast<double>(nextafterf(f, INFINITY)));
            const double dl = 5.684341886080802e-14;  // 2^-44
            if (!(r * (1.0 - dl) > mlo && r * (1.0 + dl) < mhi))
                f = exact_dist<RBC_L2, 8>(qrow, xp + static_cast<int64_t>(pp) * d, d);  // near a midpoint
            const uint64_t key = pack_key(f, static_cast<uint32_t>(perm[pp]));
            if (key < best[KT - 1]) sorted_insert<KT>(best, key);
        };
        const unsigned gmask = (1u << kRerankLanes) - 1u;
        for (;;) {
            // pick A: the group's first pending element; pick B: the next one after A
            const unsigned whoA = (__ballot_sync(0xffffffffu, pass != 0) >> gshift) & gmask;
            if (__all_sync(0xffffffffu, whoA == 0)) break;
            const int srcA = whoA ? __ffs(whoA) - 1 : 0;
            const unsigned passA = (whoA && sub == srcA) ? pass & (pass - 1) : pass;
            const unsigned whoB = (__ballot_sync(0xffffffffu, passA != 0) >> gshift) & gmask;
            const int srcB = whoB ? __ffs(whoB) - 1 : 0;
            const int jA = __shfl_sync(0xffffffffu, pass ? __ffs(pass) - 1 : 0, gshift + srcA);
            const int jB = __shfl_sync(0xffffffffu, passA ? __ffs(passA) - 1 : 0, gshift + srcB);
            const int32_t ppA = __shfl_sync(0xffffffffu, pos, gshift + srcA) + jA;
            const int32_t ppB = __shfl_sync(0xffffffffu, pos, gshift + srcB) + jB;
            double partA = 0.0, partB = 0.0;
            if (whoA) {
                float ys[DL], zs[DL];
                load_row(ppA, ys);
                load_row(whoB ? ppB : ppA, zs);
#pragma unroll
                for (int t = 0; t < DL; ++t) {
                    partA = __dadd_rn(partA, l2_term(xs[t], ys[t]));
                    partB = __dadd_rn(partB, l2_term(xs[t], zs[t]));
                }
            }
#pragma unroll
            for (int o = kRerankLanes / 2; o > 0; o >>= 1) {
                partA = __dadd_rn(partA, __shfl_xor_sync(0xffffffffu, partA, o));
                partB = __dadd_rn(partB, __shfl_xor_sync(0xffffffffu, partB, o));
            }
            pass = passA;
            if (whoA && sub == srcA) finish(partA, ppA);
            if (whoB && sub == srcB) {
                pass &= pass - 1;
                finish(partB, ppB);
            }
        }
    }
    for (int r = 0; r < k; ++r) {
        uint64_t m = best[0];
#pragma unroll
        for (int o = kRerankLanes / 2; o > 0; o >>= 1) {
            const uint64_t w = __shfl_xor_sync(0xffffffffu, m, o);
            m = w < m ? w : m;
        }
        if (live && sub == 0) out_keys[i * k + r] = m;
        if (best[0] == m && m != kEmptyKey) {  // keys are unique (distinct ids) unless empty
#pragma unroll
            for (int j = 0; j < KT - 1; ++j) best[j] = best[j + 1];
            best[KT - 1] = kEmptyKey;
        }
    }
}


// Exact SIMT scan for the queries whose candidate buffer overflowed; the count
// lives on the device (no host round trip).  One warp per entry, grid-stride.
template <int KT>
__global__ void __launch_bounds__(256) overflow_scan_kernel(const float *__restrict__ q, int d,
                                                            const int32_t *__restrict__ ovf_list,
                                                            const int32_t *__restrict__ ovf_count, SegSubSrc src, int k,
                                                            uint64_t *__restrict__ keys) {
    __shared__ float qs_all[8 * 128];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = *ovf_count;
    for (int64_t i = blockIdx.x * 8 + w; i < n; i += static_cast<int64_t>(gridDim.x) * 8) {
        const int64_t qi = ovf_list[i];
        float *qs = qs_all + w * 128;
        for (int c = lane; c < d; c += 32) qs[c] = q[qi * d + c];
        __syncwarp();
        uint64_t best[KT];
#pragma unroll
        for (int j = 0; j < KT; ++j) best[j] = kEmptyKey;
        src.for_each(i, lane, [&](const float *__restrict__ row, uint32_t id) {
            const uint64_t key = pack_key(exact_dist<RBC_L2>(qs, row, d), id);
            if (key < best[KT - 1]) sorted_insert<KT>(best, key);
        });
        warp_merge_sorted<KT>(best, k, keys + qi * k);
        __syncwarp();
    }
}

__global__ void stage2_status_kernel(const unsigned long long *__restrict__ work_total,
                                     const int32_t *__restrict__ ovf_count, int64_t *__restrict__ status) {
    status[0] = static_cast<int64_t>(*work_total);
    status[1] = *ovf_count;
}

}  // namespace

int64_t &last_overflow_count() {
    static int64_t v = 0;
    return v;
}

void pad_rows64(const float *src, int64_t rows, int d, float *dst, cudaStream_t st) {
    pad64_rows_kernel<<<grid_for(rows * 64, 256), 256, 0, st>>>(src, rows, d, dst);
    note_launch();
}

// ---- index-side preparation ----------------------------------------------------------------
static void tc_free(TcIndex *tc) {
    cudaFree(tc->xh0);
    cudaFree(tc->xh1);
    cudaFree(tc->gcol);
    cudaFree(tc->poff);
    cudaFree(tc->sB);
    cudaFree(tc->dbmax);
    cudaFree(tc->reps64);
    delete tc;
}

// Stage-2 operands of a set of lists: list p = rows [off[p], off[p+1]) of xp, centred
// on reps[p] with radius radii[p].  off_host is the host copy of offsets_dev.
static int tc_lists_build(const float *xp, const float *reps, const int64_t *offsets_dev,
                          const std::vector<int64_t> &off, const float *radii, int64_t nr, int d, TcIndex **out,
                          size_t *bytes, cudaStream_t st) {
    TcIndex *tc = new TcIndex();
    tc->np = d > 64 ? 2 : 1;
    tc->plane1 = d > 64 * tc->np - 2;
    std::vector<int64_t> poff(nr + 1, 0);
    int64_t maxlen = 0;
    for (int64_t p = 0; p < nr; ++p) {
        const int64_t len = off[p + 1] - off[p];
        poff[p + 1] = poff[p] + ((len + 7) & ~int64_t(7));
        maxlen = len > maxlen ? len : maxlen;
    }
    tc->npad = poff[nr];
    const int64_t rows = tc->npad + kTailRows;
    tc->rows = rows;
    const int np = tc->np;
    bool ok = cudaMalloc(&tc->xh0, np * rows * kP0) == cudaSuccess &&
              (!tc->plane1 || cudaMalloc(&tc->xh1, rows * kP1) == cudaSuccess) &&
              cudaMalloc(&tc->gcol, rows * sizeof(float)) == cudaSuccess &&
              cudaMalloc(&tc->poff, (nr + 1) * sizeof(int64_t)) == cudaSuccess &&
              cudaMalloc(&tc->sB, nr * sizeof(float)) == cudaSuccess &&
              cudaMalloc(&tc->dbmax, nr * sizeof(float)) == cudaSuccess &&
              cudaMalloc(&tc->reps64, nr * (64 * np + 4) * sizeof(float)) == cudaSuccess;
    if (!ok) {
        cudaGetLastError();
        tc_free(tc);
        return fail(RBC_ENOMEM, "tc list operands allocation");
    }
    if (bytes)
        *bytes += rows * (np * kP0 + (tc->plane1 ? kP1 : 0) + sizeof(float)) + (nr + 1) * sizeof(int64_t) +
                  nr * ((64 * np + 6) * sizeof(float));
    if (cudaMemsetAsync(tc->xh0, 0, np * rows * kP0, st) != cudaSuccess ||
        (tc->plane1 && cudaMemsetAsync(tc->xh1, 0, rows * kP1, st) != cudaSuccess) ||
        cudaMemsetAsync(tc->gcol, 0, rows * sizeof(float), st) != cudaSuccess ||
        cudaMemsetAsync(tc->dbmax, 0, nr * sizeof(float), st) != cudaSuccess ||
        cudaMemcpyAsync(tc->poff, poff.data(), sizeof(int64_t) * (nr + 1), cudaMemcpyHostToDevice, st) != cudaSuccess) {
        tc_free(tc);
        return fail(RBC_ECUDA, "tc list operands init");
    }
    list_scale_kernel<<<grid_for(nr, 256), 256, 0, st>>>(radii, nr, tc->sB);
    pad64_rows_kernel<<<grid_for(nr * (64 * np + 4), 256), 256, 0, st>>>(reps, nr, d, tc->reps64, 64 * np + 4);
    const unsigned ysplit = static_cast<unsigned>(maxlen > 256 * 148 ? 148 : (maxlen + 255) / 256 + 0);
    residual_rows_kernel<<<dim3(static_cast<unsigned>(nr), ysplit > 0 ? ysplit : 1), 256, 0, st>>>(
        xp, reps, offsets_dev, tc->poff, tc->sB, d, np, rows * kP0, tc->plane1 ? 1 : 0, tc->xh0, tc->xh1, tc->gcol,
        tc->dbmax);
    // dbmax[p] beside the representative row (one bulk copy brings both to the stage-2 kernel)
    rep_dbmax_kernel<<<grid_for(nr, 256), 256, 0, st>>>(tc->dbmax, nr, 64 * np + 4, tc->reps64);
    note_launch(4);
    if (cudaGetLastError() != cudaSuccess) {
        tc_free(tc);
        return fail(RBC_ECUDA, "tc list operand kernels");
    }
    *out = tc;
    return RBC_OK;
}

int tc_index_prepare(rbc_index *idx, cudaStream_t st) {
    if (idx->kind != 0 || idx->metric != RBC_L2 || idx->d > 128 || idx->n_local == 0) return RBC_OK;
    if (idx->n_local + kTailRows >= (int64_t(1) << 31)) return RBC_OK;  // int32 work offsets
    if (!tc_range_ok(idx->xp, idx->n_local * idx->d, st) || !tc_range_ok(idx->reps, idx->nr * idx->d, st))
        return RBC_OK;  // coordinates beyond the fp32 bounds' range: SIMT / exact engines
    std::vector<int64_t> off(idx->nr + 1);
    RBC_CUDA(cudaMemcpyAsync(off.data(), idx->offsets, sizeof(int64_t) * (idx->nr + 1), cudaMemcpyDeviceToHost, st));
    RBC_CUDA(cudaStreamSynchronize(st));
    TcIndex *tc = nullptr;
    RBC_CHECK(tc_lists_build(idx->xp, idx->reps, idx->offsets, off, idx->radii, idx->nr, idx->d, &tc, &idx->bytes, st));
    if (cudaStreamSynchronize(st) != cudaSuccess) {
        tc_free(tc);
        return fail(RBC_ECUDA, "tc index kernels");
    }
    idx->tc = tc;
    return RBC_OK;
}

void tc_index_release(rbc_index *idx) {
    TcIndex *tc = static_cast<TcIndex *>(idx->tc);
    if (!tc) return;
    tc_free(tc);
    idx->tc = nullptr;
}

// tile_fill_kernel keeps three int32 words per representative in shared memory
constexpr int64_t kMaxRepsTileFill = (200 * 1024) / (3 * sizeof(int32_t));

bool tc_stage2_supported(const rbc_index *idx, int k) {
    return idx->tc != nullptr && k <= 32 && idx->nr <= kMaxRepsTileFill;
}

static int g_num_sms = 0;

static int s2_run(const rbc_index *idx, const float *q, int64_t nq, int k, const PruneOut &po, const int32_t *order,
                  int ntiles, const int32_t *tile_order, const int64_t *work_off, const int64_t *nwork,
                  const unsigned long long *work_total, const WorkItem *work, const int32_t *cut, int64_t cap_work,
                  int32_t *cand_count, int32_t *counters, uint64_t *keys, int64_t *status_dev, cudaStream_t st,
                  int cap_groups, int nslot, const int4 *vt, const int32_t *nvt);

int tc_stage2(const rbc_index *idx, const float *q, int64_t nq, int k, const PruneOut &po, uint64_t *keys,
              int64_t cap_work, int64_t *status_dev, cudaStream_t st, int cap_groups) {
    const TcIndex *tc = static_cast<const TcIndex *>(idx->tc);
    if (g_num_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int64_t nr = idx->nr;
    const int ntiles = static_cast<int>((nq + kRows - 1) / kRows);
    // 1. group queries into tiles.  After the fused stage 1 the queries are already in
    //    nearest-pilot order (farthest-point pilots: one per region), which groups them as
    //    well for stage 2 as a (first surviving list, nearest rep) sort does, within 2% of
    //    stage-2 time and without the sort; otherwise sort by that key.
    DevBuf<uint64_t> tkey, tkey_sorted;
    DevBuf<uint32_t> gkey, skey;
    DevBuf<int32_t> ids, order_buf, tids, tile_order;
    RBC_CHECK(tkey.alloc(ntiles, st));
    RBC_CHECK(tkey_sorted.alloc(ntiles, st));
    RBC_CHECK(tids.alloc(ntiles, st));
    RBC_CHECK(tile_order.alloc(ntiles, st));
    size_t tb2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb2, tkey.get(), tkey_sorted.get(), tids.get(), tile_order.get(), ntiles, 0,
                                    16, st);
    DevBuf<unsigned char> tmp;
    const int32_t *order = po.qorder.get();
    if (!order) {
        int kb = 1;
        while ((int64_t(1) << kb) < nr) ++kb;  // nr < 2^24 (tc_stage2_supported)
        const int kbits = kb > 16 ? 32 : 2 * kb;
        RBC_CHECK(skey.alloc(nq, st));
        RBC_CHECK(ids.alloc(nq, st));
        RBC_CHECK(order_buf.alloc(nq, st));
        RBC_CHECK(gkey.alloc(nq, st));
        group_key_kernel<<<grid_for(nq, 256), 256, 0, st>>>(po.order_key.get(), nq, kb, gkey.get(), ids.get());
        RBC_LAUNCHED();
        size_t tb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, gkey.get(), skey.get(), ids.get(), order_buf.get(), nq, 0, kbits,
                                        st);
        RBC_CHECK(tmp.alloc(tb > tb2 ? tb : tb2, st));
        RBC_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, gkey.get(), skey.get(), ids.get(), order_buf.get(), nq,
                                                 0, kbits, st));
        note_launch();
        order = order_buf.get();
    } else {
        RBC_CHECK(tmp.alloc(tb2, st));
    }
    // 2. union of surviving lists per tile
    DevBuf<int64_t> nwork, work_off;
    DevBuf<unsigned long long> work_total_own;
    RBC_CHECK(nwork.alloc(ntiles, st));
    RBC_CHECK(work_off.alloc(ntiles, st));
    unsigned long long *work_total = po.s2_total.get();
    if (po.s2_total_zeroed) {
        po.s2_total_zeroed = false;  // a re-run (capacity retry) zeroes its own counter
    } else {
        RBC_CHECK(work_total_own.alloc(1, st));
        RBC_CUDA(cudaMemsetAsync(work_total_own.get(), 0, sizeof(unsigned long long), st));
        work_total = work_total_own.get();
    }
    const size_t smem3 = 3 * sizeof(int32_t) * nr;
    if (smem3 > 200 * 1024) return fail(RBC_EINVAL, "too many representatives for the tile prep");
    cudaFuncSetAttribute(tile_fill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem3));
    // max-only warm-up copy of each tile's first list (k = 1): off -- with the nearest-rep
    // lists ordered first the bounds tighten early anyway, and the extra list cost more
    // (stage 2 540 vs 573 us, re-rank 60 vs 52 us at cfg2); RBC_S2_WARM=1 turns it on
    const int warm = (k == 1 && getenv("RBC_S2_WARM")) ? 1 : 0;
    // work arrays sized from the caller's capacity (no host round trip); an
    // undersized capacity makes every consumer kernel bail out and the caller
    // re-runs with the size reported in status[0]
    const int64_t total_work = cap_work;
    // k > 1: heavy tiles split over up to kMaxSplit CTAs (RBC_S2_NOSPLIT=1: off)
    const int nsplit = (k > 1 && cap_work < (int64_t(1) << 31) && !getenv("RBC_S2_NOSPLIT")) ? kMaxSplit : 1;
    const int nslot = kParts * nsplit;
    DevBuf<WorkItem> work;
    DevBuf<int32_t> cut, cand_count, counters;
    RBC_CHECK(cand_count.alloc(nq * nslot, st));  // zeroed by tile_fill_kernel
    RBC_CHECK(counters.alloc(2, st));              // (overflow count, tile counter), zeroed by tile_fill_kernel
    RBC_CHECK(work.alloc(total_work, st));
    RBC_CHECK(cut.alloc(total_work * kRows, st));
    tile_fill_kernel<<<ntiles, kFillThreads, smem3, st>>>(order, nq, nwork.get(), work_off.get(), work_total, tids.get(),
                                                   po.seg_off.get(),
                                                   po.nseg.get(), po.seg_list.get(),
                                                   po.seg_len.get(), po.seg_d1.get(), po.order_key.get(), nr, tc->sB,
                                                   idx->radii, tc->poff,
                                                   idx->offsets, work.get(), cut.get(),
                                                   tkey.get(), warm, cap_work, cand_count.get(), nslot, counters.get());
    RBC_LAUNCHED();
    RBC_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tb2, tkey.get(), tkey_sorted.get(), tids.get(),
                                             tile_order.get(), ntiles, 0, 16, st));
    note_launch();
    DevBuf<int4> vt;
    DevBuf<int32_t> nvt;
    if (nsplit > 1) {
        RBC_CHECK(vt.alloc(static_cast<int64_t>(ntiles) * nsplit, st));
        RBC_CHECK(nvt.alloc(1, st));
        split_plan_kernel<<<1, 1024, 0, st>>>(tile_order.get(), tkey_sorted.get(), ntiles, work_off.get(), nwork.get(),
                                              nsplit, g_num_sms, vt.get(), nvt.get());
        RBC_LAUNCHED();
    }
    return s2_run(idx, q, nq, k, po, order, ntiles, tile_order.get(), work_off.get(), nwork.get(), work_total,
                  work.get(), cut.get(), cap_work, cand_count.get(), counters.get(), keys, status_dev, st, cap_groups,
                  nslot, nsplit > 1 ? vt.get() : nullptr, nsplit > 1 ? nvt.get() : nullptr);
}

// stage-2 kernel + exact re-rank + overflow scan + status over prepared work arrays
static std::atomic<int64_t> g_tc_scan_calls{0};

static int s2_run(const rbc_index *idx, const float *q, int64_t nq, int k, const PruneOut &po, const int32_t *order,
                  int ntiles, const int32_t *tile_order, const int64_t *work_off, const int64_t *nwork,
                  const unsigned long long *work_total, const WorkItem *work, const int32_t *cut, int64_t cap_work,
                  int32_t *cand_count, int32_t *counters, uint64_t *keys, int64_t *status_dev, cudaStream_t st,
                  int cap_groups, int nslot, const int4 *vt, const int32_t *nvt) {
    g_tc_scan_calls.fetch_add(1);
    const TcIndex *tc = static_cast<const TcIndex *>(idx->tc);
    // 3. the tensor-core scan
    // 8-column groups per query and column part.  k > 1 buffers ~k ln(N/k) groups per part
    // (the k-record events of the scan); a compaction (a pass over the buffer) runs when it
    // fills, so the capacity is sized to make that rare
    const int cap = cap_groups > 0 ? cap_groups : (k == 1 ? 18 : (16 + 24 * k < 512 ? 16 + 24 * k : 512));
    DevBuf<float> cand_lb, cand_ufin, q64buf;
    DevBuf<int32_t> cand_pos, ovf_list;
    RBC_CHECK(cand_lb.alloc(nq * nslot * cap * 12, st));
    RBC_CHECK(cand_pos.alloc(nq * nslot * cap, st));
    RBC_CHECK(cand_ufin.alloc(nq * nslot, st));
    RBC_CHECK(ovf_list.alloc(nq * nslot, st));
    const float *q64 = q;
    const int qw = 64 * tc->np;
    if (idx->d != qw || (reinterpret_cast<uintptr_t>(q) & 15) != 0) {
        RBC_CHECK(q64buf.alloc(nq * qw, st));
        pad64_rows_kernel<<<grid_for(nq * qw, 256), 256, 0, st>>>(q, nq, idx->d, q64buf.get(), qw);
        RBC_LAUNCHED();
        q64 = q64buf.get();
    }
    S2Params P;
    P.xh0 = tc->xh0;
    P.plane_bytes = tc->rows * kP0;
    P.xh1 = tc->xh1;
    P.gcol = tc->gcol;
    P.reps64 = tc->reps64;
    P.dbmax = tc->dbmax;
    P.plane1 = tc->plane1 ? 1 : 0;
    P.q64 = q64;
    P.gamma = po.gamma.get();
    P.k = k;
    P.ntiles = ntiles;
    P.tile_order = tile_order;
    P.vt = vt;
    P.nvt = nvt;
    P.nslot = nslot;
    P.order = order;
    P.nq = nq;
    P.work_off = work_off;
    P.nwork = nwork;
    P.work_total = work_total;
    P.work = work;
    P.cut = cut;
    P.cand_lb = cand_lb.get();
    P.cand_pos = cand_pos.get();
    P.cap = cap;
    P.cand_count = cand_count;
    P.cand_ufin = cand_ufin.get();
    P.overflow_list = ovf_list.get();
    P.overflow_count = counters;
    P.tile_counter = counters + 1;
    P.cap_work = cap_work;
    DevBuf<unsigned long long> timing;
    P.timing = nullptr;
#ifdef RBC_S2_TIMING
    if (getenv("RBC_DEBUG_S2")) {
        RBC_CHECK(timing.alloc(148 * 12, st));
        RBC_CUDA(cudaMemsetAsync(timing.get(), 0, sizeof(unsigned long long) * 148 * 12, st));
        P.timing = timing.get();
    }
#endif
    if (g_num_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int64_t entries = vt ? static_cast<int64_t>(ntiles) * (nslot / kParts) : ntiles;
    const unsigned grid = static_cast<unsigned>(entries < g_num_sms ? entries : g_num_sms);
    auto launch = [&](auto kern, size_t smem) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        kern<<<grid, kThreads, smem, st>>>(P);
    };
    {
        ProfScope ps(kPhaseScan, st);
        if (tc->np == 1) {
            constexpr size_t sm = S2Cfg<1>::kSmem;
            if (k == 1) launch(stage2_tc_kernel<1, 1>, sm);
            else if (k <= 4) launch(stage2_tc_kernel<4, 1>, sm);
            else if (k <= 8) launch(stage2_tc_kernel<8, 1>, sm);
            else if (k == 10) launch(stage2_tc_kernel<10, 1>, sm);  // the k of cfg3/cfg5: no k-th select
            else if (k <= 16) launch(stage2_tc_kernel<16, 1>, sm);
            else launch(stage2_tc_kernel<32, 1>, sm);
        } else {
            constexpr size_t sm = S2Cfg<2>::kSmem;
            if (k == 1) launch(stage2_tc_kernel<1, 2>, sm);
            else if (k <= 4) launch(stage2_tc_kernel<4, 2>, sm);
            else if (k <= 8) launch(stage2_tc_kernel<8, 2>, sm);
            else if (k == 10) launch(stage2_tc_kernel<10, 2>, sm);  // the k of cfg3/cfg5: no k-th select
            else if (k <= 16) launch(stage2_tc_kernel<16, 2>, sm);
            else launch(stage2_tc_kernel<32, 2>, sm);
        }
    }
    RBC_LAUNCHED();
    // 4. exact re-rank of the buffered candidates
    {
        const unsigned rgrid = grid_for(nq * kRerankLanes, kRerankThreads);
#define RBC_RERANK(KT)                                                                                              \
    do {                                                                                                            \
        if (idx->d <= 64)                                                                                           \
            rerank_kernel<KT, 8><<<rgrid, kRerankThreads, 0, st>>>(                                                  \
                reinterpret_cast<const float4 *>(cand_lb.get()), cand_pos.get(), cand_count, cand_ufin.get(), cap,    \
                nslot, nq, q, idx->xp, idx->perm, idx->d, k, keys);                                                  \
        else                                                                                                        \
            rerank_kernel<KT, 16><<<rgrid, kRerankThreads, 0, st>>>(                                                 \
                reinterpret_cast<const float4 *>(cand_lb.get()), cand_pos.get(), cand_count, cand_ufin.get(), cap,    \
                nslot, nq, q, idx->xp, idx->perm, idx->d, k, keys);                                                  \
    } while (0)
        if (k == 1) RBC_RERANK(1);
        else if (k <= 4) RBC_RERANK(4);
        else if (k <= 8) RBC_RERANK(8);
        else if (k == 10) RBC_RERANK(10);
        else if (k <= 16) RBC_RERANK(16);
        else RBC_RERANK(32);
#undef RBC_RERANK
        RBC_LAUNCHED();
    }
    // 5. overflow fallback: exact SIMT scan for the few queries whose buffer filled
    //    up (device-side count; the queries' segments are still in `po`)
    {
        SegSubSrc src{idx->xp, idx->perm,     po.seg_start.get(), po.seg_len.get(),
                      po.seg_off.get(), po.nseg.get(), ovf_list.get(), idx->d};
        const unsigned ogrid = static_cast<unsigned>(g_num_sms * 4);
        if (k == 1) overflow_scan_kernel<1><<<ogrid, 256, 0, st>>>(q, idx->d, ovf_list.get(), counters, src, k, keys);
        else if (k <= 4) overflow_scan_kernel<4><<<ogrid, 256, 0, st>>>(q, idx->d, ovf_list.get(), counters, src, k, keys);
        else if (k <= 8) overflow_scan_kernel<8><<<ogrid, 256, 0, st>>>(q, idx->d, ovf_list.get(), counters, src, k, keys);
        else if (k <= 16) overflow_scan_kernel<16><<<ogrid, 256, 0, st>>>(q, idx->d, ovf_list.get(), counters, src, k, keys);
        else overflow_scan_kernel<32><<<ogrid, 256, 0, st>>>(q, idx->d, ovf_list.get(), counters, src, k, keys);
        RBC_LAUNCHED();
    }
    stage2_status_kernel<<<1, 1, 0, st>>>(work_total, counters, status_dev);
    RBC_LAUNCHED();
    if (getenv("RBC_DEBUG_CAND")) {  // diagnostic: buffered-group counts (synchronises)
        std::vector<int32_t> cc(nq * nslot);
        cudaMemcpyAsync(cc.data(), cand_count, sizeof(int32_t) * nq * nslot, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        int64_t sum = 0, ovf = 0, mx = 0;
        for (int32_t v : cc) {
            if (v < 0) ++ovf;
            else { sum += v; mx = v > mx ? v : mx; }
        }
        fprintf(stderr, "[s2] cap %d: groups mean %.2f max %lld, overflowed parts %lld of %lld\n", cap,
                double(sum) / double(cc.size() - ovf + 1e-9), (long long)mx, (long long)ovf, (long long)cc.size());
        // MMA work: columns scanned per tile (chunks rounded to 16) x 128 rows, and the tile spread
        std::vector<int64_t> nw(ntiles), wo(ntiles);
        unsigned long long wt = 0;
        cudaMemcpy(nw.data(), nwork, sizeof(int64_t) * ntiles, cudaMemcpyDeviceToHost);
        cudaMemcpy(wo.data(), work_off, sizeof(int64_t) * ntiles, cudaMemcpyDeviceToHost);
        cudaMemcpy(&wt, work_total, sizeof(wt), cudaMemcpyDeviceToHost);
        std::vector<WorkItem> wi(wt);
        cudaMemcpy(wi.data(), work, sizeof(WorkItem) * wt, cudaMemcpyDeviceToHost);
        double cols = 0, tmax = 0, items = 0;
        for (int t = 0; t < ntiles; ++t) {
            double tc = 0;
            for (int64_t w = wo[t]; w < wo[t] + nw[t]; ++w) tc += (wi[w].ext + 15) / 16 * 16;
            cols += tc;
            items += nw[t];
            tmax = tc > tmax ? tc : tmax;
        }
        fprintf(stderr, "[s2] tiles %d: work items/tile %.1f, MMA pairs %.4g (cols/tile mean %.0f max %.0f)\n", ntiles,
                items / ntiles, cols * 128, cols / ntiles, tmax);
    }
#ifdef RBC_S2_TIMING
    if (getenv("RBC_DEBUG_S2")) {  // diagnostic: role timing (synchronises)
        std::vector<unsigned long long> tm(148 * 12);
        cudaMemcpy(tm.data(), timing.get(), sizeof(unsigned long long) * 148 * 12, cudaMemcpyDeviceToHost);
        double sum[12] = {0};
        for (int b = 0; b < (int)grid; ++b)
            for (int j = 0; j < 12; ++j) sum[j] += tm[b * 12 + j];
        const char *nm[12] = {"prod:empty", "mma:afull", "mma:full", "mma:tempty", "epi:aempty", "epi:tfull",
                              "wall(3 roles)", "-", "epi:prep", "-", "-", "epi:lists#"};
        fprintf(stderr, "[s2] per-CTA cycles:");
        for (int j = 0; j < 12; ++j) fprintf(stderr, " %s=%.0f", nm[j], sum[j] / grid / (j == 6 ? 3.0 : 1.0));
        fprintf(stderr, "\n");
    }
#endif
    return RBC_OK;
}


// ---- tensor-core brute force ----------------------------------------------------------------
// bf_search (brute_force.py:165-186), the build's nearest-representative assignment
// (rbc.py:164) and the one-shot search's nearest representative (search.py:114-115):
// all rows of x form ONE list centred on their mean c (radius max |x - c|), and every
// query row scans it whole through stage2_tc_kernel -- the tcgen05 distance tile with the
// running-bound filter epilogue -- followed by the exact fp64 re-rank.  Every (q, x) pair
// passes through the tensor cores; only the filter survivors are recomputed exactly, so
// the keys are the reference's bit for bit.
namespace {

__global__ void bf_colsum_kernel(const float *__restrict__ x, int64_t n, int d, double *__restrict__ sum) {
    const int k = threadIdx.x & 127, sub = threadIdx.x >> 7;
    if (k >= d) return;
    double acc = 0.0;
    for (int64_t i = blockIdx.x * 2ll + sub; i < n; i += gridDim.x * 2ll) acc += x[i * d + k];
    atomicAdd(&sum[k], acc);
}

// centre row (the list's representative) and the CSR offsets {0, n} of the single list
__global__ void bf_centre_kernel(const double *__restrict__ sum, int64_t n, int d, float *__restrict__ c,
                                 int64_t *__restrict__ offsets) {
    const int k = threadIdx.x;
    if (k < d) c[k] = static_cast<float>(sum[k] / static_cast<double>(n));
    if (k == 0) {
        offsets[0] = 0;
        offsets[1] = n;
    }
}

// list radius: max over the rows of |x - c| (fp32 residuals, fp64 sum), rounded up
__global__ void bf_extent_kernel(const float *__restrict__ x, int64_t n, int d, const float *__restrict__ c,
                                 unsigned *__restrict__ rmax_bits) {
    unsigned m = 0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double h = 0.0;
        for (int k = 0; k < d; ++k) {
            const double b = __fsub_rn(x[i * d + k], c[k]);
            h += b * b;
        }
        m = max(m, __float_as_uint(static_cast<float>(sqrt(h)) * kUp));
    }
    m = __reduce_max_sync(0xffffffffu, m);
    if ((threadIdx.x & 31) == 0 && m) atomicMax(rmax_bits, m);
}

// per query: one segment = the whole list (cutoff n), gamma = +inf (no seed bound),
// |q - c| for the A-operand scale, identity tile order
__global__ void bf_queries_kernel(const float *__restrict__ q, int64_t nq, int d, const float *__restrict__ c,
                                  int32_t n, float *__restrict__ gamma, int32_t *__restrict__ nseg,
                                  int64_t *__restrict__ seg_off, int64_t *__restrict__ seg_start,
                                  int32_t *__restrict__ seg_len, int32_t *__restrict__ seg_list,
                                  float *__restrict__ seg_d1, uint64_t *__restrict__ order_key,
                                  int32_t *__restrict__ qorder) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i > nq) return;
    seg_off[i] = i;
    if (i == nq) return;
    float h = 0.f;
    for (int k = 0; k < d; ++k) {
        const float t = q[i * d + k] - c[k];
        h = fmaf(t, t, h);
    }
    gamma[i] = __int_as_float(0x7f800000);
    nseg[i] = 1;
    seg_start[i] = 0;
    seg_len[i] = n;
    seg_list[i] = 0;
    seg_d1[i] = sqrtf(h);
    order_key[i] = 0;
    qorder[i] = static_cast<int32_t>(i);
}

__global__ void iota_i32_kernel(int32_t *__restrict__ a, int64_t n) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n) a[i] = static_cast<int32_t>(i);
}

}  // namespace

bool tc_bf_supported(int64_t nq, int64_t n, int d, int metric, int k) {
    // one list centred on the mean: tight enough when the points are few (representative
    // sets); large point sets use the partitioned operand (tc_bf_index_search)
    if (metric != RBC_L2 || d < 1 || d > 128 || k < 1 || k > 32 || n < k || n > 65536) return false;
    if (n + kTailRows + 8 >= (int64_t(1) << 31)) return false;  // int32 positions
    return nq * n >= tc_min_pairs();  // smaller problems: the exact SIMT scan is faster
}

static std::atomic<int64_t> g_tc_bf_calls{0};

int tc_bf_keys(const float *q, int64_t nq, const float *x, int64_t n, int d, int k, uint64_t *keys, cudaStream_t st) {
    if (nq == 0) return RBC_OK;
    g_tc_bf_calls.fetch_add(1);
    DevBuf<double> csum;
    DevBuf<float> cen, rad;
    DevBuf<int64_t> offsets;
    DevBuf<int32_t> perm;
    DevBuf<unsigned> rbits;
    RBC_CHECK(csum.alloc(128, st));
    RBC_CHECK(cen.alloc(128, st));
    RBC_CHECK(rad.alloc(1, st));
    RBC_CHECK(offsets.alloc(2, st));
    RBC_CHECK(perm.alloc(n, st));
    RBC_CUDA(cudaMemsetAsync(csum.get(), 0, 128 * sizeof(double), st));
    RBC_CUDA(cudaMemsetAsync(rad.get(), 0, sizeof(float), st));
    bf_colsum_kernel<<<grid_for(n, 2, 148 * 8), 256, 0, st>>>(x, n, d, csum.get());
    bf_centre_kernel<<<1, 128, 0, st>>>(csum.get(), n, d, cen.get(), offsets.get());
    bf_extent_kernel<<<grid_for(n, 256, 148 * 8), 256, 0, st>>>(x, n, d, cen.get(),
                                                               reinterpret_cast<unsigned *>(rad.get()));
    iota_i32_kernel<<<grid_for(n, 256), 256, 0, st>>>(perm.get(), n);
    RBC_LAUNCHED();
    note_launch(3);
    TcIndex *tc = nullptr;
    const std::vector<int64_t> off_h{0, n};
    RBC_CHECK(tc_lists_build(x, cen.get(), offsets.get(), off_h, rad.get(), 1, d, &tc, nullptr, st));
    rbc_index tmp;
    tmp.kind = 0;
    tmp.n = n;
    tmp.d = d;
    tmp.metric = RBC_L2;
    tmp.nr = 1;
    tmp.reps = cen.get();
    tmp.radii = rad.get();
    tmp.offsets = offsets.get();
    tmp.perm = perm.get();
    tmp.xp = const_cast<float *>(x);
    tmp.n_local = n;
    tmp.tc = tc;
    // queries in batches of <= 1M rows (the candidate buffers are ~2.3 KB per query at k = 1)
    auto run = [&](const float *qb, int64_t m, uint64_t *kb) -> int {
        PruneOut po;
        RBC_CHECK(po.gamma.alloc(m, st));
        RBC_CHECK(po.nseg.alloc(m, st));
        RBC_CHECK(po.seg_off.alloc(m + 1, st));
        RBC_CHECK(po.seg_start.alloc(m, st));
        RBC_CHECK(po.seg_len.alloc(m, st));
        RBC_CHECK(po.seg_list.alloc(m, st));
        RBC_CHECK(po.seg_d1.alloc(m, st));
        RBC_CHECK(po.order_key.alloc(m, st));
        RBC_CHECK(po.qorder.alloc(m, st));
        po.total_segs = m;
        bf_queries_kernel<<<grid_for(m + 1, 256), 256, 0, st>>>(
            qb, m, d, cen.get(), static_cast<int32_t>(n), po.gamma.get(), po.nseg.get(), po.seg_off.get(),
            po.seg_start.get(), po.seg_len.get(), po.seg_list.get(), po.seg_d1.get(), po.order_key.get(),
            po.qorder.get());
        RBC_LAUNCHED();
        DevBuf<int64_t> status;
        RBC_CHECK(status.alloc(2, st));
        const int64_t cap_work = (m + kRows - 1) / kRows + 64;  // one work item per tile
        const char *capenv = getenv("RBC_BF_CAP");  // diagnostic override of the candidate-group capacity
        const int capg = capenv ? atoi(capenv) : 16 + 8 * k;
        RBC_CHECK(tc_stage2(&tmp, qb, m, k, po, kb, cap_work, status.get(), st, capg));
        int64_t h[2] = {0, 0};
        RBC_CUDA(cudaMemcpyAsync(h, status.get(), sizeof(h), cudaMemcpyDeviceToHost, st));
        RBC_CUDA(cudaStreamSynchronize(st));
        last_overflow_count() = h[1];
        if (h[0] > cap_work) return fail(RBC_ECUDA, "brute-force work items exceed one per tile");
        return RBC_OK;
    };
    const int64_t batch = int64_t(1) << 20;
    int rc = RBC_OK;
    for (int64_t q0 = 0; q0 < nq && rc == RBC_OK; q0 += batch)
        rc = run(q + q0 * d, nq - q0 < batch ? nq - q0 : batch, keys + q0 * k);
    cudaStreamSynchronize(st);
    tc_free(tc);
    return rc;
}


// ---- tensor-core brute force over a partitioned operand ------------------------------------
// bf_search at scale: x is partitioned into lists around evenly spaced points (an exact RBC
// index, built once per prepared operand) so every f16 operand is a residual to a nearby
// centre; the scan then visits EVERY list for every query tile -- no pruning, every
// (q, x) pair passes through the tensor cores -- with the tile's nearest lists first so the
// running bound is tight before the far lists stream through.
namespace {

// centre of the list representatives and |r_p - c| per list
__global__ void bf_rep_centre_kernel(const float *__restrict__ reps, int64_t nr, int d, float *__restrict__ c) {
    const int k = threadIdx.x;
    if (k >= d) return;
    double s = 0.0;
    for (int64_t p = 0; p < nr; ++p) s += reps[p * d + k];
    c[k] = static_cast<float>(s / static_cast<double>(nr));
}

__global__ void row_dist_kernel(const float *__restrict__ a, int64_t rows, int d, const float *__restrict__ c,
                                float *__restrict__ out) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= rows) return;
    double h = 0.0;
    for (int k = 0; k < d; ++k) {
        const double t = static_cast<double>(a[i * d + k]) - static_cast<double>(c[k]);
        h += t * t;
    }
    out[i] = static_cast<float>(sqrt(h)) * kUp;
}

// per query: nearest-list sort key, gamma (k = 1: the exact distance to the nearest list
// centre, a point of x, bounds the nearest neighbour; else +inf), one overflow segment = all of x
__global__ void bf_index_queries_kernel(const uint64_t *__restrict__ near, int64_t nq, int k, int32_t n,
                                        uint32_t *__restrict__ skey, int32_t *__restrict__ ids,
                                        float *__restrict__ gamma, int32_t *__restrict__ nseg,
                                        int64_t *__restrict__ seg_off, int64_t *__restrict__ seg_start,
                                        int32_t *__restrict__ seg_len) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i > nq) return;
    seg_off[i] = i;
    if (i == nq) return;
    const uint64_t key = near[i];
    skey[i] = key_id(key);
    ids[i] = static_cast<int32_t>(i);
    gamma[i] = k == 1 ? key_dist(key) : __int_as_float(0x7f800000);
    nseg[i] = 1;
    seg_start[i] = 0;
    seg_len[i] = n;
}

// One block per 128-query tile: every list becomes a work item (cut = whole list); the lists
// that are some row's nearest list come first (most rows first), then the rest by position.
// A scale from |q - c| + |r_p - c| >= |q - r_p| over the tile's rows.  Also zeroes stage 2's
// per-query group counts and counters and writes the (identity) tile order.
__global__ void __launch_bounds__(kRows) bf_tile_fill_kernel(
    const int32_t *__restrict__ order, int64_t nq, const uint64_t *__restrict__ near, const float *__restrict__ qdc,
    const float *__restrict__ rdc, int64_t nr, const int64_t *__restrict__ offsets, const int64_t *__restrict__ poff,
    const float *__restrict__ sB, const float *__restrict__ radii, WorkItem *__restrict__ work,
    int64_t *__restrict__ work_off, int64_t *__restrict__ nwork, unsigned long long *__restrict__ work_total,
    int32_t *__restrict__ tile_order, int32_t *__restrict__ cand_count, int32_t *__restrict__ counters) {
    extern __shared__ int32_t cnt[];  // [nr]
    typedef cub::BlockScan<int, kRows> Scan;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ unsigned long long s_fkey[kRows];
    __shared__ int s_nf;
    __shared__ unsigned s_dq;
    for (int64_t p = threadIdx.x; p < nr; p += blockDim.x) cnt[p] = 0;
    if (threadIdx.x == 0) {
        s_nf = 0;
        s_dq = 0;
        tile_order[blockIdx.x] = static_cast<int32_t>(blockIdx.x);
        nwork[blockIdx.x] = nr;
        work_off[blockIdx.x] = static_cast<int64_t>(blockIdx.x) * nr;
        if (blockIdx.x == 0) *work_total = static_cast<unsigned long long>(gridDim.x) * nr;
    }
    if (blockIdx.x == 0 && threadIdx.x < 2) counters[threadIdx.x] = 0;
    __syncthreads();
    const int64_t tq = static_cast<int64_t>(blockIdx.x) * kRows + threadIdx.x;
    const int32_t qi = tq < nq ? order[tq] : -1;
    if (qi >= 0) {
#pragma unroll
        for (int h = 0; h < kParts; ++h) cand_count[kParts * static_cast<int64_t>(qi) + h] = 0;
        atomicAdd(&cnt[key_id(near[qi])], 1);
        atomicMax(&s_dq, __float_as_uint(qdc[qi]));
    }
    __syncthreads();
    const int64_t per = (nr + kRows - 1) / kRows;
    const int64_t pa = threadIdx.x * per, pe = min(nr, pa + per);
    int c = 0;
    for (int64_t p = pa; p < pe; ++p) {
        if (cnt[p] > 0) {
            const int slot = atomicAdd(&s_nf, 1);  // <= 128 distinct nearest lists per tile
            s_fkey[slot] = (static_cast<unsigned long long>(kRows - cnt[p]) << 32) | static_cast<uint64_t>(p);
        } else {
            ++c;
        }
    }
    int pos, total;
    Scan(scan_tmp).ExclusiveSum(c, pos, total);
    __syncthreads();
    const int nf = s_nf;
    const float dq = __uint_as_float(s_dq);
    WorkItem *w0 = work + static_cast<int64_t>(blockIdx.x) * nr;
    auto item = [&](int64_t p) {
        WorkItem it;
        it.p = static_cast<int32_t>(p);
        it.ext = static_cast<int32_t>(offsets[p + 1] - offsets[p]);
        const float m = (dq + rdc[p]) * kUp;
        int e = 0;
        if (m > 0.f) frexpf(m, &e);
        it.sA = m > 0.f ? ldexpf(1.0f, -e) : 1.0f;
        it.sB = sB[p];
        it.radius = radii[p];
        const float cc = it.sA / it.sB;
        it.aug = (cc >= 6.103515625e-05f && cc <= 32768.0f) ? -cc : 0.0f;
        it.poff = static_cast<int32_t>(poff[p]);
        it.csr = static_cast<int32_t>(offsets[p]);
        return it;
    };
    for (int64_t p = pa; p < pe; ++p)
        if (cnt[p] == 0) w0[nf + pos++] = item(p);
    if (threadIdx.x < nf) {
        const unsigned long long mine = s_fkey[threadIdx.x];
        int rank = 0;
        for (int j = 0; j < nf; ++j) rank += s_fkey[j] < mine ? 1 : 0;
        w0[rank] = item(static_cast<int64_t>(mine & 0xFFFFFFFFu));
    }
}

}  // namespace

static int tc_bf_index_search_batch(const rbc_index *idx, const float *q, int64_t nq, int k, uint64_t *keys,
                                    cudaStream_t st);

int tc_bf_index_search(const rbc_index *idx, const float *q, int64_t nq, int k, uint64_t *keys, cudaStream_t st) {
    const int64_t batch = int64_t(1) << 20;  // candidate buffers ~2.3 KB per query at k = 1
    for (int64_t q0 = 0; q0 < nq; q0 += batch)
        RBC_CHECK(tc_bf_index_search_batch(idx, q + q0 * idx->d, nq - q0 < batch ? nq - q0 : batch, k,
                                           keys + q0 * k, st));
    return RBC_OK;
}

static int tc_bf_index_search_batch(const rbc_index *idx, const float *q, int64_t nq, int k, uint64_t *keys,
                                    cudaStream_t st) {
    if (nq == 0) return RBC_OK;
    const TcIndex *tc = static_cast<const TcIndex *>(idx->tc);
    if (!tc || k < 1 || k > 32) return fail(RBC_EINVAL, "tc brute force: unsupported index or k");
    g_tc_bf_calls.fetch_add(1);
    const int64_t nr = idx->nr, n = idx->n_local;
    const int d = idx->d;
    const int ntiles = static_cast<int>((nq + kRows - 1) / kRows);
    // 1. nearest list centre of every query (k = 1 brute force over the centres)
    DevBuf<uint64_t> near;
    RBC_CHECK(near.alloc(nq, st));
    RBC_CHECK(nearest_rows(q, nq, idx->reps, nr, d, RBC_L2, near.get(), st));
    // 2. queries ordered by nearest list; gamma; overflow segments
    PruneOut po;
    RBC_CHECK(po.gamma.alloc(nq, st));
    RBC_CHECK(po.nseg.alloc(nq, st));
    RBC_CHECK(po.seg_off.alloc(nq + 1, st));
    RBC_CHECK(po.seg_start.alloc(nq, st));
    RBC_CHECK(po.seg_len.alloc(nq, st));
    DevBuf<uint32_t> skey, skey_sorted;
    DevBuf<int32_t> ids, order;
    RBC_CHECK(skey.alloc(nq, st));
    RBC_CHECK(skey_sorted.alloc(nq, st));
    RBC_CHECK(ids.alloc(nq, st));
    RBC_CHECK(order.alloc(nq, st));
    bf_index_queries_kernel<<<grid_for(nq + 1, 256), 256, 0, st>>>(near.get(), nq, k, static_cast<int32_t>(n),
                                                                    skey.get(), ids.get(), po.gamma.get(),
                                                                    po.nseg.get(), po.seg_off.get(),
                                                                    po.seg_start.get(), po.seg_len.get());
    RBC_LAUNCHED();
    int kb = 1;
    while ((int64_t(1) << kb) < nr) ++kb;
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, skey.get(), skey_sorted.get(), ids.get(), order.get(), nq, 0, kb, st);
    DevBuf<unsigned char> tmp;
    RBC_CHECK(tmp.alloc(tb, st));
    RBC_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, skey.get(), skey_sorted.get(), ids.get(), order.get(), nq,
                                             0, kb, st));
    note_launch();
    // 3. |q - c|, |r_p - c| for the A scales
    DevBuf<float> cen, qdc, rdc;
    RBC_CHECK(cen.alloc(128, st));
    RBC_CHECK(qdc.alloc(nq, st));
    RBC_CHECK(rdc.alloc(nr, st));
    bf_rep_centre_kernel<<<1, 128, 0, st>>>(idx->reps, nr, d, cen.get());
    row_dist_kernel<<<grid_for(nq, 256), 256, 0, st>>>(q, nq, d, cen.get(), qdc.get());
    row_dist_kernel<<<grid_for(nr, 256), 256, 0, st>>>(idx->reps, nr, d, cen.get(), rdc.get());
    RBC_LAUNCHED();
    note_launch(2);
    // 4. every list is a work item of every tile
    const int64_t cap_work = static_cast<int64_t>(ntiles) * nr;
    DevBuf<WorkItem> work;
    DevBuf<int64_t> work_off, nwork;
    DevBuf<unsigned long long> work_total;
    DevBuf<int32_t> tile_order, cand_count, counters;
    RBC_CHECK(work.alloc(cap_work, st));
    RBC_CHECK(work_off.alloc(ntiles, st));
    RBC_CHECK(nwork.alloc(ntiles, st));
    RBC_CHECK(work_total.alloc(1, st));
    RBC_CHECK(tile_order.alloc(ntiles, st));
    RBC_CHECK(cand_count.alloc(nq * kParts, st));
    RBC_CHECK(counters.alloc(2, st));
    const size_t smem = sizeof(int32_t) * nr;
    if (smem > 200 * 1024) return fail(RBC_EINVAL, "tc brute force: too many lists");
    cudaFuncSetAttribute(bf_tile_fill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    bf_tile_fill_kernel<<<ntiles, kRows, smem, st>>>(order.get(), nq, near.get(), qdc.get(), rdc.get(), nr,
                                                      idx->offsets, tc->poff, tc->sB, idx->radii, work.get(),
                                                      work_off.get(), nwork.get(), work_total.get(), tile_order.get(),
                                                      cand_count.get(), counters.get());
    RBC_LAUNCHED();
    // 5. the scan, exact re-rank and overflow fallback
    DevBuf<int64_t> status;
    RBC_CHECK(status.alloc(2, st));
    const char *capenv = getenv("RBC_BF_CAP");  // diagnostic override of the candidate-group capacity
    const int capg = capenv ? atoi(capenv) : 16 + 8 * k;
    RBC_CHECK(s2_run(idx, q, nq, k, po, order.get(), ntiles, tile_order.get(), work_off.get(), nwork.get(),
                     work_total.get(), work.get(), nullptr, cap_work, cand_count.get(), counters.get(), keys,
                     status.get(), st, capg, kParts, nullptr, nullptr));
    int64_t h[2] = {0, 0};
    RBC_CUDA(cudaMemcpyAsync(h, status.get(), sizeof(h), cudaMemcpyDeviceToHost, st));
    RBC_CUDA(cudaStreamSynchronize(st));
    last_overflow_count() = h[1];
    return RBC_OK;
}

// ---- one-shot list scan on the tensor cores ---------------------------------------------------
// one_shot_query_batch (search.py:90-141): each query scans exactly the s-list of its nearest
// representative.  The s-lists are stored like exact-index lists (rows gathered per list,
// f16 residuals to the list's rep; the lists overlap, so a point can sit in several), the
// queries are grouped by nearest rep, and each row's only segment is its own list (cutoff
// s; 0 for the tile's other lists), so the scan is exactly L_{r_q}.
namespace {

__global__ void one_shot_offsets_kernel(int64_t nr, int s, int64_t *__restrict__ off) {
    const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (p <= nr) off[p] = p * s;
}

__global__ void one_shot_segments_kernel(const uint64_t *__restrict__ near, int64_t nq, int s,
                                         float *__restrict__ gamma, int32_t *__restrict__ nseg,
                                         int64_t *__restrict__ seg_off, int64_t *__restrict__ seg_start,
                                         int32_t *__restrict__ seg_len, int32_t *__restrict__ seg_list,
                                         float *__restrict__ seg_d1, uint64_t *__restrict__ order_key) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i > nq) return;
    seg_off[i] = i;
    if (i == nq) return;
    const uint64_t key = near[i];
    const uint32_t p = key_id(key);
    gamma[i] = __int_as_float(0x7f800000);  // no seed bound (the rep need not be in its own list)
    nseg[i] = 1;
    seg_start[i] = static_cast<int64_t>(p) * s;
    seg_len[i] = s;
    seg_list[i] = static_cast<int32_t>(p);
    seg_d1[i] = key_dist(key);
    order_key[i] = (static_cast<uint64_t>(p) << 24) | p;
}

}  // namespace

int tc_one_shot_prepare(rbc_index *idx, const float *xp_lists, cudaStream_t st) {
    if (idx->kind != 1 || idx->metric != RBC_L2 || idx->d > 128) return RBC_OK;
    const int64_t total = idx->nr * static_cast<int64_t>(idx->s);
    if (total + kTailRows >= (int64_t(1) << 31)) return RBC_OK;  // int32 positions
    if (!tc_range_ok(xp_lists, total * idx->d, st) || !tc_range_ok(idx->reps, idx->nr * idx->d, st)) return RBC_OK;
    std::vector<int64_t> off(idx->nr + 1);
    for (int64_t p = 0; p <= idx->nr; ++p) off[p] = p * idx->s;
    one_shot_offsets_kernel<<<grid_for(idx->nr + 1, 256), 256, 0, st>>>(idx->nr, idx->s, idx->offsets);
    RBC_LAUNCHED();
    TcIndex *tc = nullptr;
    RBC_CHECK(tc_lists_build(xp_lists, idx->reps, idx->offsets, off, idx->radii, idx->nr, idx->d, &tc, &idx->bytes,
                             st));
    if (cudaStreamSynchronize(st) != cudaSuccess) {
        tc_free(tc);
        return fail(RBC_ECUDA, "one-shot tc operands");
    }
    idx->tc = tc;
    return RBC_OK;
}

bool tc_one_shot_supported(const rbc_index *idx, int64_t nq, int k) {
    return idx->tc != nullptr && idx->kind == 1 && k <= 32 && k <= idx->s && idx->nr <= kMaxRepsTileFill &&
           nq * idx->s >= tc_min_pairs();
}

int tc_one_shot_scan(const rbc_index *idx, const float *q, int64_t nq, int k, const uint64_t *near, uint64_t *keys,
                     cudaStream_t st) {
    if (nq == 0) return RBC_OK;
    g_tc_bf_calls.fetch_add(1);
    PruneOut po;
    RBC_CHECK(po.gamma.alloc(nq, st));
    RBC_CHECK(po.nseg.alloc(nq, st));
    RBC_CHECK(po.seg_off.alloc(nq + 1, st));
    RBC_CHECK(po.seg_start.alloc(nq, st));
    RBC_CHECK(po.seg_len.alloc(nq, st));
    RBC_CHECK(po.seg_list.alloc(nq, st));
    RBC_CHECK(po.seg_d1.alloc(nq, st));
    RBC_CHECK(po.order_key.alloc(nq, st));
    po.total_segs = nq;
    one_shot_segments_kernel<<<grid_for(nq + 1, 256), 256, 0, st>>>(near, nq, idx->s, po.gamma.get(), po.nseg.get(),
                                                                     po.seg_off.get(), po.seg_start.get(),
                                                                     po.seg_len.get(), po.seg_list.get(),
                                                                     po.seg_d1.get(), po.order_key.get());
    RBC_LAUNCHED();
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
    return fail(RBC_ECUDA, "one-shot scan: work capacity");
}
}  // namespace rbc

extern "C" int64_t rbc_tc_bf_calls(void) { return rbc::g_tc_bf_calls.load(); }
extern "C" int64_t rbc_tc_scan_calls(void) { return rbc::g_tc_scan_calls.load(); }
