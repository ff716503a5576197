// build.cu -- representative sampling and the two index builds.
//
//  * bernoulli_pcg64: numpy's PCG64 stream reproduced on device (rbc.py:57-59).
//    Thread t owns draws [t*C, (t+1)*C): it jumps the 128-bit LCG to draw t*C
//    (O(log n) multiply-adds), then steps sequentially; flags are compacted
//    in id order (np.flatnonzero).
//  * build_exact (rbc.py:147-180): nearest-rep assignment as a k=1 scan of X
//    against R (exact keys, lowest rep position on ties), then ONE stable
//    radix sort on (owner << 32 | f32 bits(dist)) with the point id as
//    payload, which reproduces lexsort((id, dist, owner)) (rbc.py:168),
//    then segment offsets by binary search and radii = segment tails.
//  * build_one_shot (rbc.py:183-200): the s nearest points of every rep.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "common.cuh"
#include "kernels.cuh"
#include "tc_scan.cuh"

namespace rbc {

typedef unsigned __int128 u128;

__device__ __forceinline__ u128 pcg_mult() {
    return (static_cast<u128>(0x2360ED051FC65DA4ull) << 64) | static_cast<u128>(0x4385DF649FCCF645ull);
}

__device__ __forceinline__ uint64_t xsl_rr(u128 s) {
    const uint64_t hi = static_cast<uint64_t>(s >> 64), lo = static_cast<uint64_t>(s);
    const uint64_t v = hi ^ lo;
    const unsigned rot = static_cast<unsigned>(hi >> 58);
    return (v >> rot) | (v << ((64u - rot) & 63u));
}

// state after `delta` LCG steps (standard PCG jump-ahead)
__device__ __forceinline__ u128 pcg_advance(u128 state, u128 inc, uint64_t delta) {
    u128 acc_mult = 1, acc_plus = 0, cur_mult = pcg_mult(), cur_plus = inc;
    while (delta > 0) {
        if (delta & 1) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    return acc_mult * state + acc_plus;
}

constexpr int kDrawsPerThread = 64;

__global__ void bernoulli_flags_kernel(int64_t n, double p, uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi,
                                       uint64_t inc_lo, uint8_t *__restrict__ flags) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int64_t i0 = t * kDrawsPerThread;
    if (i0 >= n) return;
    const u128 inc = (static_cast<u128>(inc_hi) << 64) | inc_lo;
    u128 s = pcg_advance((static_cast<u128>(st_hi) << 64) | st_lo, inc, static_cast<uint64_t>(i0));
    const u128 mult = pcg_mult();
    const int64_t i1 = i0 + kDrawsPerThread < n ? i0 + kDrawsPerThread : n;
    for (int64_t i = i0; i < i1; ++i) {
        s = s * mult + inc;
        const double u = static_cast<double>(xsl_rr(s) >> 11) * (1.0 / 9007199254740992.0);
        flags[i] = u < p ? 1 : 0;
    }
}

int bernoulli(int64_t n, double p, uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t *ids_out,
              int64_t *count_host, cudaStream_t st) {
    DevBuf<uint8_t> flags;
    DevBuf<int64_t> count;
    RBC_CHECK(flags.alloc(n, st));
    RBC_CHECK(count.alloc(1, st));
    bernoulli_flags_kernel<<<grid_for((n + kDrawsPerThread - 1) / kDrawsPerThread, 256), 256, 0, st>>>(
        n, p, st_hi, st_lo, inc_hi, inc_lo, flags.get());
    RBC_LAUNCHED();
    thrust::counting_iterator<int64_t> it(0);
    size_t tb = 0;
    cub::DeviceSelect::Flagged(nullptr, tb, it, flags.get(), ids_out, count.get(), n, st);
    DevBuf<unsigned char> tmp;
    RBC_CHECK(tmp.alloc(tb, st));
    RBC_CUDA(cub::DeviceSelect::Flagged(tmp.get(), tb, it, flags.get(), ids_out, count.get(), n, st));
    note_launch();
    RBC_CUDA(cudaMemcpyAsync(count_host, count.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    RBC_CUDA(cudaStreamSynchronize(st));
    return RBC_OK;
}

// ---- build_exact -------------------------------------------------------------
__global__ void gather_rows_kernel(const float *__restrict__ x, const int64_t *__restrict__ ids, int64_t rows, int d,
                                   float *__restrict__ out) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < rows * d;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[t] = x[ids[t / d] * d + t % d];
}

int gather_rows(const float *x, const int64_t *ids, int64_t rows, int d, float *out, cudaStream_t st) {
    if (rows == 0) return RBC_OK;
    gather_rows_kernel<<<grid_for(rows * d, 256, 148 * 64), 256, 0, st>>>(x, ids, rows, d, out);
    RBC_LAUNCHED();
    return RBC_OK;
}

// (owner, dist) -> assignment key (dist bits << 32 | rep pos)
__global__ void pack_assign_kernel(const int64_t *__restrict__ owner, const float *__restrict__ dist, int64_t m,
                                   uint64_t *__restrict__ assign) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < m) assign[i] = pack_key(dist[i], static_cast<uint32_t>(owner[i]));
}

// assignment key (dist bits, rep pos) -> sort key (rep pos << 32 | dist bits), payload id
__global__ void owner_sort_keys_kernel(const uint64_t *__restrict__ assign, int64_t n, uint64_t *__restrict__ keys,
                                       uint32_t *__restrict__ vals) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const uint64_t a = assign[i];
    keys[i] = (static_cast<uint64_t>(key_id(a)) << 32) | (a >> 32);
    vals[i] = static_cast<uint32_t>(i);
}

__global__ void finish_lists_kernel(const uint64_t *__restrict__ skeys, const uint32_t *__restrict__ svals, int64_t n,
                                    int64_t *__restrict__ list_ids, float *__restrict__ list_dists) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    list_ids[i] = svals[i];
    list_dists[i] = __uint_as_float(static_cast<uint32_t>(skeys[i]));
}

// offsets[p] = first sorted position whose owner >= p; radii[p] = tail dist
__global__ void segment_offsets_kernel(const uint64_t *__restrict__ skeys, int64_t n, int64_t nr,
                                       int64_t *__restrict__ offsets, float *__restrict__ radii) {
    const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (p > nr) return;
    auto lower = [&](uint64_t target) {
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (skeys[mid] < target) lo = mid + 1;
            else hi = mid;
        }
        return lo;
    };
    const int64_t a = lower(static_cast<uint64_t>(p) << 32);
    offsets[p] = a;
    if (p < nr) {
        const int64_t b = lower(static_cast<uint64_t>(p + 1) << 32);
        radii[p] = b > a ? __uint_as_float(static_cast<uint32_t>(skeys[b - 1])) : 0.f;
    }
}

int build_exact(const float *x, int64_t n, int d, int metric, const int64_t *rep_ids, int64_t nr, int64_t *list_ids,
                int64_t *offsets, float *list_dists, float *radii, cudaStream_t st) {
    DevBuf<float> reps;
    DevBuf<uint64_t> assign, keys, skeys;
    DevBuf<uint32_t> vals, svals;
    RBC_CHECK(reps.alloc(nr * d, st));
    RBC_CHECK(assign.alloc(n, st));
    RBC_CHECK(gather_rows(x, rep_ids, nr, d, reps.get(), st));
    // nearest representative of every point: key64 argmin over rep positions
    RBC_CHECK(nearest_rows(x, n, reps.get(), nr, d, metric, assign.get(), st));
    RBC_CHECK(keys.alloc(n, st));
    RBC_CHECK(skeys.alloc(n, st));
    RBC_CHECK(vals.alloc(n, st));
    RBC_CHECK(svals.alloc(n, st));
    owner_sort_keys_kernel<<<grid_for(n, 256), 256, 0, st>>>(assign.get(), n, keys.get(), vals.get());
    RBC_LAUNCHED();
    int owner_bits = 1;
    while ((int64_t(1) << owner_bits) < nr) ++owner_bits;
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.get(), skeys.get(), vals.get(), svals.get(), n, 0,
                                    32 + owner_bits, st);
    DevBuf<unsigned char> tmp;
    RBC_CHECK(tmp.alloc(tb, st));
    RBC_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, keys.get(), skeys.get(), vals.get(), svals.get(), n, 0,
                                             32 + owner_bits, st));
    note_launch();
    finish_lists_kernel<<<grid_for(n, 256), 256, 0, st>>>(skeys.get(), svals.get(), n, list_ids, list_dists);
    RBC_LAUNCHED();
    segment_offsets_kernel<<<grid_for(nr + 1, 256), 256, 0, st>>>(skeys.get(), n, nr, offsets, radii);
    RBC_LAUNCHED();
    return RBC_OK;
}

// ---- build_one_shot ------------------------------------------------------------
__global__ void one_shot_finish_kernel(const uint64_t *__restrict__ keys, int64_t nr, int s,
                                       int64_t *__restrict__ lists, float *__restrict__ radii) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t >= nr * s) return;
    const uint64_t key = keys[t];
    lists[t] = key_id(key);
    if (t % s == s - 1) radii[t / s] = key_dist(key);
}

int build_one_shot(const float *x, int64_t n, int d, int metric, const int64_t *rep_ids, int64_t nr, int s,
                   int64_t *lists, float *radii, cudaStream_t st) {
    DevBuf<float> reps;
    DevBuf<uint64_t> keys;
    RBC_CHECK(reps.alloc(nr * d, st));
    RBC_CHECK(keys.alloc(nr * s, st));
    RBC_CHECK(gather_rows(x, rep_ids, nr, d, reps.get(), st));
    // the s nearest points of every rep: bf_search(reps, X, s) (rbc.py:196-200) through the
    // brute-force dispatch (tensor cores / SIMT filter / exact)
    RBC_CHECK(bf_search_keys(reps.get(), nr, x, n, d, metric, s, keys.get(), st));
    one_shot_finish_kernel<<<grid_for(nr * s, 256), 256, 0, st>>>(keys.get(), nr, s, lists, radii);
    RBC_LAUNCHED();
    return RBC_OK;
}


// ---- lists of a representative shard from received (owner, dist) entries ----------------------
// The sharded build (distributed.py build_exact_distributed): every rank assigns its slice
// of X, the entries travel to the rank owning their representative, and each rank sorts
// what it received.  Entries arrive in increasing id order (contiguous id slices,
// concatenated in rank order), so one stable sort on (owner << 32 | f32 bits(dist))
// reproduces lexsort((id, dist, owner)) (rbc.py:168) for the owned lists.
int build_local_lists(const int64_t *owner, const float *dist, int64_t m, int64_t nr, int64_t *order,
                      int64_t *offsets, float *sorted_dists, cudaStream_t st) {
    DevBuf<uint64_t> assign, keys, skeys;
    DevBuf<uint32_t> vals, svals;
    DevBuf<float> radii;
    RBC_CHECK(assign.alloc(m, st));
    RBC_CHECK(keys.alloc(m, st));
    RBC_CHECK(skeys.alloc(m, st));
    RBC_CHECK(vals.alloc(m, st));
    RBC_CHECK(svals.alloc(m, st));
    RBC_CHECK(radii.alloc(nr, st));
    if (m > 0) {
        pack_assign_kernel<<<grid_for(m, 256), 256, 0, st>>>(owner, dist, m, assign.get());
        RBC_LAUNCHED();
        owner_sort_keys_kernel<<<grid_for(m, 256), 256, 0, st>>>(assign.get(), m, keys.get(), vals.get());
        RBC_LAUNCHED();
        int owner_bits = 1;
        while ((int64_t(1) << owner_bits) < nr) ++owner_bits;
        size_t tb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.get(), skeys.get(), vals.get(), svals.get(), m, 0,
                                        32 + owner_bits, st);
        DevBuf<unsigned char> tmp;
        RBC_CHECK(tmp.alloc(tb, st));
        RBC_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, keys.get(), skeys.get(), vals.get(), svals.get(), m, 0,
                                                 32 + owner_bits, st));
        note_launch();
        finish_lists_kernel<<<grid_for(m, 256), 256, 0, st>>>(skeys.get(), svals.get(), m, order, sorted_dists);
        RBC_LAUNCHED();
    }
    segment_offsets_kernel<<<grid_for(nr + 1, 256), 256, 0, st>>>(skeys.get(), m, nr, offsets, radii.get());
    RBC_LAUNCHED();
    return RBC_OK;
}

// radii[p] = max(radii[p], dist of every entry owned by p) (dist >= 0: float bits order)
__global__ void list_radii_kernel(const int64_t *__restrict__ owner, const float *__restrict__ dist, int64_t m,
                                  float *__restrict__ radii) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < m) atomicMax(reinterpret_cast<unsigned *>(radii) + owner[i], __float_as_uint(dist[i]));
}

int local_list_radii(const int64_t *owner, const float *dist, int64_t m, int64_t nr, float *radii, cudaStream_t st) {
    RBC_CUDA(cudaMemsetAsync(radii, 0, sizeof(float) * nr, st));
    if (m == 0) return RBC_OK;
    list_radii_kernel<<<grid_for(m, 256), 256, 0, st>>>(owner, dist, m, radii);
    RBC_LAUNCHED();
    return RBC_OK;
}
}  // namespace rbc
