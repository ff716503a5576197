// prune_math.cuh -- the reference's pruning predicates, bit-faithful (float64).
#pragma once

#include "common.cuh"

namespace rbc {

// #entries of an ascending f32 list <= thr, compared in f64 (search.py:77-82)
__device__ __forceinline__ int32_t list_cutoff_dev(const float *__restrict__ l, int32_t m, double thr) {
    int32_t lo = 0, hi = m;
    while (lo < hi) {
        const int32_t mid = (lo + hi) >> 1;
        if (static_cast<double>(l[mid]) <= thr) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// search.py:62-74, evaluated in f64 exactly as numpy does
__device__ __forceinline__ bool survives(float dist, float radius, double g) {
    const double dd = dist, r = radius;
    return (dd <= 3.0 * g) && ((dd < __dadd_rn(g, r)) || (dd <= g));
}

// search.py:194: pruned by the radius test
__device__ __forceinline__ bool pruned_radius(float dist, float radius, double g) {
    const double dd = dist;
    return dd >= __dadd_rn(g, static_cast<double>(radius)) && dd > g;
}

// search.py:195: pruned by the 3 gamma test
__device__ __forceinline__ bool pruned_3gamma(float dist, double g) { return static_cast<double>(dist) > 3.0 * g; }

}  // namespace rbc
