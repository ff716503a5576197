// common.cuh -- shared device helpers for the B200 RBC kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/rbc_b200.h"

namespace rbc {

constexpr uint64_t kEmptyKey = ~0ull;

// ---- error plumbing --------------------------------------------------------
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);
void note_launch(int n = 1);

// ---- optional per-phase CUDA-event timing (rbc_profile_*) ------------------
enum Phase { kPhaseStage1 = 0, kPhasePrune = 1, kPhaseStage2 = 2, kPhaseBuild = 3, kPhaseScan = 4, kNumPhases = 8 };
void prof_mark(int phase, bool begin, cudaStream_t st);
struct ProfScope {
    int phase;
    cudaStream_t st;
    ProfScope(int p, cudaStream_t s) : phase(p), st(s) { prof_mark(phase, true, st); }
    ~ProfScope() { prof_mark(phase, false, st); }
};

#define RBC_CUDA(call)                                                                          \
    do {                                                                                        \
        cudaError_t _e = (call);                                                                \
        if (_e != cudaSuccess)                                                                  \
            return ::rbc::fail(RBC_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e));  \
    } while (0)

#define RBC_LAUNCHED()                                                                          \
    do {                                                                                        \
        ::rbc::note_launch();                                                                   \
        cudaError_t _e = cudaGetLastError();                                                    \
        if (_e != cudaSuccess)                                                                  \
            return ::rbc::fail(RBC_ECUDA, std::string("launch: ") + cudaGetErrorString(_e));    \
    } while (0)

#define RBC_CHECK(expr)                                                                         \
    do {                                                                                        \
        int _rc = (expr);                                                                       \
        if (_rc != RBC_OK) return _rc;                                                          \
    } while (0)

// Keep freed blocks in the device's default stream-ordered pool (otherwise
// every synchronisation returns them to the OS and the next search re-maps
// hundreds of MB).
void retain_pool_memory();

// Scratch arena for captured (CUDA-graph) searches: while a thread has an arena
// installed, DevBuf carves its buffers out of it (fixed addresses, no frees), so
// the whole stream-ordered sequence can be captured once and replayed.  With
// `base == nullptr` the arena only measures the bytes a search requests.
struct Arena {
    char *base = nullptr;
    size_t cap = 0;
    size_t used = 0;
};
Arena *&current_arena();

// Stream-ordered scratch allocation (cudaMallocAsync pool, or the current arena).
template <typename T>
struct DevBuf {
    T *ptr = nullptr;
    cudaStream_t stream = nullptr;
    bool owned = false;
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    ~DevBuf() {
        if (ptr && owned) cudaFreeAsync(ptr, stream);
    }
    int alloc(size_t count, cudaStream_t s) {
        stream = s;
        if (count == 0) count = 1;
        Arena *a = current_arena();
        if (a && a->base) {
            const size_t bytes = (count * sizeof(T) + 255) & ~size_t(255);
            if (a->used + bytes > a->cap) return fail(RBC_ENOMEM, "search arena exhausted");
            ptr = reinterpret_cast<T *>(a->base + a->used);
            a->used += bytes;
            owned = false;
            return RBC_OK;
        }
        if (a) a->used += (count * sizeof(T) + 255) & ~size_t(255);  // measuring pass
        owned = true;
        retain_pool_memory();
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(&ptr), count * sizeof(T), s);
        if (e != cudaSuccess) {
            ptr = nullptr;
            cudaGetLastError();
            return fail(RBC_ENOMEM, std::string("cudaMallocAsync: ") + cudaGetErrorString(e));
        }
        return RBC_OK;
    }
    T *get() const { return ptr; }
};

inline unsigned grid_for(int64_t work, int per_block, int64_t cap = (1 << 30)) {
    int64_t g = (work + per_block - 1) / per_block;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return static_cast<unsigned>(g);
}

// ---- the reference distance arithmetic (metric.py:36-54) -------------------
// fp32 inputs widened to fp64; k-sequential accumulation; __dmul_rn/__dadd_rn
// forbid FMA contraction so the result is bit-identical to the scalar
// mulsd/addsd loop numba emits; one rounding to fp32 at the end.
__device__ __forceinline__ double l2_term(float a, float b) {
    double diff = __dsub_rn(static_cast<double>(a), static_cast<double>(b));
    return __dmul_rn(diff, diff);
}
__device__ __forceinline__ double l1_term(float a, float b) {
    return fabs(__dsub_rn(static_cast<double>(a), static_cast<double>(b)));
}

template <int METRIC>
__device__ __forceinline__ double exact_acc4(double acc, const float4 &x, const float4 &y) {
    acc = __dadd_rn(acc, METRIC == RBC_L2 ? l2_term(x.x, y.x) : l1_term(x.x, y.x));
    acc = __dadd_rn(acc, METRIC == RBC_L2 ? l2_term(x.y, y.y) : l1_term(x.y, y.y));
    acc = __dadd_rn(acc, METRIC == RBC_L2 ? l2_term(x.z, y.z) : l1_term(x.z, y.z));
    acc = __dadd_rn(acc, METRIC == RBC_L2 ? l2_term(x.w, y.w) : l1_term(x.w, y.w));
    return acc;
}

// B4 = float4 loads of each row in flight per step (4: 16 coordinates; 8 for
// latency-bound callers with registers to spare)
template <int METRIC, int B4 = 4>
__device__ __forceinline__ float exact_dist(const float *__restrict__ a, const float *__restrict__ b, int d) {
    double acc = 0.0;
    int k = 0;
    if (((d & 3) | ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15)) == 0) {
        // 16-byte rows: 4*B4 coordinates (B4+B4 vector loads) in flight per step
        const float4 *a4 = reinterpret_cast<const float4 *>(a), *b4 = reinterpret_cast<const float4 *>(b);
        for (; k + 4 * B4 <= d; k += 4 * B4) {
            float4 x[B4], y[B4];
#pragma unroll
            for (int j = 0; j < B4; ++j) {
                x[j] = a4[(k >> 2) + j];
                y[j] = b4[(k >> 2) + j];
            }
#pragma unroll
            for (int j = 0; j < B4; ++j) acc = exact_acc4<METRIC>(acc, x[j], y[j]);
        }
        for (; k + 4 <= d; k += 4) acc = exact_acc4<METRIC>(acc, a4[k >> 2], b4[k >> 2]);
    }
    // loads batched 8 at a time (independent, in flight together); the
    // accumulation itself stays strictly in coordinate order
    for (; k + 8 <= d; k += 8) {
        float av[8], bv[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            av[j] = a[k + j];
            bv[j] = b[k + j];
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
            acc = __dadd_rn(acc, METRIC == RBC_L2 ? l2_term(av[j], bv[j]) : l1_term(av[j], bv[j]));
    }
    for (; k < d; ++k) acc = __dadd_rn(acc, METRIC == RBC_L2 ? l2_term(a[k], b[k]) : l1_term(a[k], b[k]));
    if (METRIC == RBC_L2) return __double2float_rn(__dsqrt_rn(acc));
    return __double2float_rn(acc);
}

// key64 = (f32 bits << 32) | id   (brute_force.py:62-68)
__device__ __forceinline__ uint64_t pack_key(float dist, uint32_t id) {
    return (static_cast<uint64_t>(__float_as_uint(dist)) << 32) | id;
}
__device__ __forceinline__ float key_dist(uint64_t key) { return __uint_as_float(static_cast<uint32_t>(key >> 32)); }
__device__ __forceinline__ uint32_t key_id(uint64_t key) { return static_cast<uint32_t>(key); }

__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        uint64_t w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w < v ? w : v;
    }
    return v;
}

// Sorted insertion of key into an ascending register array best[0..KT).
template <int KT>
__device__ __forceinline__ void sorted_insert(uint64_t (&best)[KT], uint64_t key) {
#pragma unroll
    for (int j = 0; j < KT; ++j) {
        uint64_t lo = best[j] < key ? best[j] : key;
        uint64_t hi = best[j] < key ? key : best[j];
        best[j] = lo;
        key = hi;
    }
}

// k smallest keys over the 32 lanes' ascending arrays -> out[0..k) (lane 0
// writes).  Each round the warp minimum of the lane heads is popped.
template <int KT>
__device__ __forceinline__ void warp_merge_sorted(uint64_t (&best)[KT], int k, uint64_t *out) {
    const int lane = threadIdx.x & 31;
    for (int r = 0; r < k; ++r) {
        uint64_t m = warp_min_u64(best[0]);
        if (lane == 0) out[r] = m;
        if (best[0] == m && m != kEmptyKey) {  // keys are unique (distinct ids) unless empty
#pragma unroll
            for (int j = 0; j < KT - 1; ++j) best[j] = best[j + 1];
            best[KT - 1] = kEmptyKey;
        }
    }
}

__device__ __forceinline__ void unpack_to(uint64_t key, int64_t *id, float *dist) {
    if (key == kEmptyKey) {
        *id = -1;
        *dist = __uint_as_float(0x7f800000u);
    } else {
        *id = static_cast<int64_t>(key_id(key));
        *dist = key_dist(key);
    }
}

}  // namespace rbc
