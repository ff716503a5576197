// abi.cu -- the extern "C" boundary (include/rbc_b200.h).
#include <cub/cub.cuh>

#include <atomic>
#include <cmath>
#include <climits>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "index.cuh"
#include "kernels.cuh"
#include "search.cuh"
#include "tc_scan.cuh"

namespace rbc {

static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string &msg) { g_last_error = msg; }
int fail(int code, const std::string &msg) {
    g_last_error = msg;
    return code;
}
void note_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
int64_t launch_count_now() { return g_launches.load(); }

Arena *&current_arena() {
    static thread_local Arena *a = nullptr;
    return a;
}

bool profiling_on();

void retain_pool_memory() {
    static thread_local int done_for = -1;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev == done_for) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    done_for = dev;
}

// per-phase event pairs, recorded on the launching stream when enabled
struct ProfRec {
    int phase;
    cudaEvent_t a, b;
};
static bool g_prof_on = false;
static std::vector<ProfRec> g_prof;
static std::vector<cudaEvent_t> g_prof_open(kNumPhases, nullptr);

bool profiling_on() { return g_prof_on; }

void prof_mark(int phase, bool begin, cudaStream_t st) {
    if (!g_prof_on) return;
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    cudaEventRecord(e, st);
    if (begin) {
        g_prof_open[phase] = e;
    } else if (g_prof_open[phase]) {
        g_prof.push_back({phase, g_prof_open[phase], e});
        g_prof_open[phase] = nullptr;
    } else {
        cudaEventDestroy(e);
    }
}

int gather_rows(const float *x, const int64_t *ids, int64_t rows, int d, float *out, cudaStream_t st);
int bernoulli(int64_t n, double p, uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t *ids_out,
              int64_t *count_host, cudaStream_t st);
int build_exact(const float *x, int64_t n, int d, int metric, const int64_t *rep_ids, int64_t nr, int64_t *list_ids,
                int64_t *offsets, float *list_dists, float *radii, cudaStream_t st);
int build_local_lists(const int64_t *owner, const float *dist, int64_t m, int64_t nr, int64_t *order,
                      int64_t *offsets, float *sorted_dists, cudaStream_t st);
int local_list_radii(const int64_t *owner, const float *dist, int64_t m, int64_t nr, float *radii, cudaStream_t st);
int build_one_shot(const float *x, int64_t n, int d, int metric, const int64_t *rep_ids, int64_t nr, int s,
                   int64_t *lists, float *radii, cudaStream_t st);

static inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// Host -> device copy of a large host buffer split over kCopyLanes concurrent
// copies (side streams ordered after `st`, joined back into `st`): several
// copies in flight keep the PCIe link busier than one.  The side streams and
// events belong to one caller object (per index, guarded by its mutex) and are
// created on the device that is current when the object is first used.
static constexpr int kCopyLanes = 4;
struct CopyLanes {
    int device = -1;
    cudaStream_t side[kCopyLanes] = {};
    cudaEvent_t ev_start = nullptr, ev_done[kCopyLanes] = {};
    void release() {
        for (int i = 0; i < kCopyLanes; ++i) {
            if (side[i]) cudaStreamDestroy(side[i]);
            if (ev_done[i]) cudaEventDestroy(ev_done[i]);
            side[i] = nullptr;
            ev_done[i] = nullptr;
        }
        if (ev_start) cudaEventDestroy(ev_start);
        ev_start = nullptr;
        device = -1;
    }
    ~CopyLanes() { release(); }
};

static int copy_h2d_split(CopyLanes *lanes, void *dst, const void *src, size_t bytes, cudaStream_t st) {
    if (lanes == nullptr || bytes < (size_t(8) << 20)) {
        RBC_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
        return RBC_OK;
    }
    int dev = 0;
    RBC_CUDA(cudaGetDevice(&dev));
    if (lanes->device != dev) {
        lanes->release();
        RBC_CUDA(cudaEventCreateWithFlags(&lanes->ev_start, cudaEventDisableTiming));
        for (int i = 0; i < kCopyLanes; ++i) {
            RBC_CUDA(cudaStreamCreateWithFlags(&lanes->side[i], cudaStreamNonBlocking));
            RBC_CUDA(cudaEventCreateWithFlags(&lanes->ev_done[i], cudaEventDisableTiming));
        }
        lanes->device = dev;
    }
    RBC_CUDA(cudaEventRecord(lanes->ev_start, st));
    const size_t part = ((bytes + kCopyLanes - 1) / kCopyLanes + 255) & ~size_t(255);
    for (int i = 0; i < kCopyLanes; ++i) {
        const size_t off = part * i;
        if (off >= bytes) break;
        const size_t len = bytes - off < part ? bytes - off : part;
        RBC_CUDA(cudaStreamWaitEvent(lanes->side[i], lanes->ev_start, 0));
        RBC_CUDA(cudaMemcpyAsync(static_cast<char *>(dst) + off, static_cast<const char *>(src) + off, len,
                                 cudaMemcpyHostToDevice, lanes->side[i]));
        RBC_CUDA(cudaEventRecord(lanes->ev_done[i], lanes->side[i]));
        RBC_CUDA(cudaStreamWaitEvent(st, lanes->ev_done[i], 0));
    }
    return RBC_OK;
}

static int check_common(int64_t n, int d, int metric) {
    if (metric != RBC_L2 && metric != RBC_L1) return fail(RBC_EINVAL, "metric must be 0 (l2) or 1 (l1)");
    if (d < 1) return fail(RBC_EINVAL, "dim must be >= 1");
    if (n < 0 || n > 0xFFFFFFFFll) return fail(RBC_EINVAL, "point count must be in [0, 2^32)");
    return RBC_OK;
}

template <typename T>
static int dalloc(T **p, size_t count, size_t &bytes) {
    if (count == 0) count = 1;
    cudaError_t e = cudaMalloc(reinterpret_cast<void **>(p), count * sizeof(T));
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(RBC_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    }
    bytes += count * sizeof(T);
    return RBC_OK;
}

__global__ void i64_to_i32_kernel(const int64_t *__restrict__ a, int64_t n, int32_t *__restrict__ b) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x)
        b[t] = static_cast<int32_t>(a[t]);
}

__global__ void gather_rows_i32_kernel(const float *__restrict__ x, const int32_t *__restrict__ ids, int64_t rows,
                                       int d, float *__restrict__ out) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < rows * d;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[t] = x[static_cast<int64_t>(ids[t / d]) * d + t % d];
}

// copy list p's segment from the full CSR into the shard CSR
__global__ void copy_segments_kernel(const int64_t *__restrict__ src_off, const int64_t *__restrict__ dst_off,
                                     const int64_t *__restrict__ list_ids, const float *__restrict__ list_dists,
                                     int32_t *__restrict__ perm, float *__restrict__ ldist) {
    const int64_t p = blockIdx.x;
    const int64_t len = dst_off[p + 1] - dst_off[p];
    for (int64_t j = threadIdx.x; j < len; j += blockDim.x) {
        perm[dst_off[p] + j] = static_cast<int32_t>(list_ids[src_off[p] + j]);
        ldist[dst_off[p] + j] = list_dists[src_off[p] + j];
    }
}

// sorted entry i of a local shard: id and row of received entry order[i]
__global__ void gather_local_kernel(const int64_t *__restrict__ order, const int64_t *__restrict__ ids,
                                    const float *__restrict__ rows, int64_t m, int d, int32_t *__restrict__ perm,
                                    float *__restrict__ xp) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < m * d;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = t / d, c = t - i * d;
        const int64_t j = order[i];
        xp[t] = rows[j * d + c];
        if (c == 0) perm[i] = static_cast<int32_t>(ids[j]);
    }
}

// [min, max] of an int64 array (index-upload validation)
__global__ void minmax_i64_kernel(const int64_t *__restrict__ a, int64_t n, unsigned long long *__restrict__ out) {
    long long lo = LLONG_MAX, hi = LLONG_MIN;
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const long long v = a[t];
        lo = v < lo ? v : lo;
        hi = v > hi ? v : hi;
    }
    // order-preserving unsigned image of the signed values
    atomicMin(&out[0], static_cast<unsigned long long>(lo) ^ 0x8000000000000000ull);
    atomicMax(&out[1], static_cast<unsigned long long>(hi) ^ 0x8000000000000000ull);
}

// every id of a[0..n) in [0, limit) (the reference's load_index / search would raise
// IndexError; on the device an out-of-range id is an out-of-bounds gather)
static int check_ids_in_range(const int64_t *a, int64_t n, int64_t limit, const char *what, cudaStream_t st) {
    if (n == 0) return RBC_OK;
    DevBuf<unsigned long long> mm;
    RBC_CHECK(mm.alloc(2, st));
    const unsigned long long init[2] = {~0ull, 0ull};
    RBC_CUDA(cudaMemcpyAsync(mm.get(), init, sizeof(init), cudaMemcpyHostToDevice, st));
    minmax_i64_kernel<<<grid_for(n, 256, 148 * 8), 256, 0, st>>>(a, n, mm.get());
    RBC_LAUNCHED();
    unsigned long long h[2] = {0, 0};
    RBC_CUDA(cudaMemcpyAsync(h, mm.get(), sizeof(h), cudaMemcpyDeviceToHost, st));
    RBC_CUDA(cudaStreamSynchronize(st));
    const long long lo = static_cast<long long>(h[0] ^ 0x8000000000000000ull);
    const long long hi = static_cast<long long>(h[1] ^ 0x8000000000000000ull);
    if (lo < 0 || hi >= limit)
        return fail(RBC_EINVAL, std::string(what) + " out of range [0, " + std::to_string(limit) + "): min " +
                                    std::to_string(lo) + ", max " + std::to_string(hi));
    return RBC_OK;
}

static int index_common(rbc_index *idx, const float *x, const int64_t *rep_ids, const float *radii, cudaStream_t st) {
    RBC_CHECK(dalloc(&idx->x, idx->n * idx->d, idx->bytes));
    RBC_CHECK(dalloc(&idx->reps, idx->nr * idx->d, idx->bytes));
    RBC_CHECK(dalloc(&idx->rep_ids, idx->nr, idx->bytes));
    RBC_CHECK(dalloc(&idx->radii, idx->nr, idx->bytes));
    RBC_CUDA(cudaMemcpyAsync(idx->x, x, sizeof(float) * idx->n * idx->d, cudaMemcpyDeviceToDevice, st));
    RBC_CUDA(cudaMemcpyAsync(idx->rep_ids, rep_ids, sizeof(int64_t) * idx->nr, cudaMemcpyDeviceToDevice, st));
    RBC_CUDA(cudaMemcpyAsync(idx->radii, radii, sizeof(float) * idx->nr, cudaMemcpyDeviceToDevice, st));
    RBC_CHECK(gather_rows(idx->x, idx->rep_ids, idx->nr, idx->d, idx->reps, st));
    RBC_CUDA(cudaGetDevice(&idx->device));
    return RBC_OK;
}

static int exact_create(const float *x, int64_t n, int32_t d, int32_t metric, const int64_t *rep_ids, int64_t nr,
                        const int64_t *list_ids, const int64_t *list_offsets, const float *list_dists,
                        const float *radii, const uint8_t *owned, rbc_index **out, cudaStream_t st) {
    RBC_CHECK(check_common(n, d, metric));
    if (nr < 1 || nr > n) return fail(RBC_EINVAL, "n_reps must be in [1, n]");
    rbc_index *idx = new rbc_index();
    idx->kind = 0;
    idx->n = n;
    idx->d = d;
    idx->metric = metric;
    idx->nr = nr;
    idx->shard = owned != nullptr;
    int rc = check_ids_in_range(rep_ids, nr, n, "rep_ids", st);
    if (rc != RBC_OK) {
        delete idx;
        return rc;
    }
    rc = index_common(idx, x, rep_ids, radii, st);
    std::vector<int64_t> off_full(nr + 1), off_local(nr + 1, 0);
    if (rc == RBC_OK) rc = dalloc(&idx->offsets, nr + 1, idx->bytes);
    if (rc == RBC_OK && cudaMemcpyAsync(off_full.data(), list_offsets, sizeof(int64_t) * (nr + 1),
                                        cudaMemcpyDeviceToHost, st) != cudaSuccess)
        rc = fail(RBC_ECUDA, "offsets D2H");
    if (rc == RBC_OK && cudaStreamSynchronize(st) != cudaSuccess) rc = fail(RBC_ECUDA, "sync");
    // the lists must partition the n points (RbcExactIndex, rbc.py:87-115): CSR offsets from
    // 0 to n, non-decreasing, every id in [0, n)
    if (rc == RBC_OK) {
        bool ok = off_full[0] == 0 && off_full[nr] == n;
        for (int64_t p = 0; ok && p < nr; ++p) ok = off_full[p + 1] >= off_full[p];
        if (!ok) rc = fail(RBC_EINVAL, "list offsets must rise from 0 to n (the lists partition the points)");
    }
    if (rc == RBC_OK) rc = check_ids_in_range(list_ids, n, n, "list ids", st);
    if (rc == RBC_OK) {
        for (int64_t p = 0; p < nr; ++p) {
            const int64_t len = off_full[p + 1] - off_full[p];
            off_local[p + 1] = off_local[p] + ((owned == nullptr || owned[p]) ? len : 0);
        }
        idx->n_local = off_local[nr];
        rc = dalloc(&idx->perm, idx->n_local, idx->bytes);
    }
    if (rc == RBC_OK) rc = dalloc(&idx->list_dists, idx->n_local, idx->bytes);
    if (rc == RBC_OK) rc = dalloc(&idx->xp, idx->n_local * d, idx->bytes);
    if (rc == RBC_OK && cudaMemcpyAsync(idx->offsets, off_local.data(), sizeof(int64_t) * (nr + 1),
                                        cudaMemcpyHostToDevice, st) != cudaSuccess)
        rc = fail(RBC_ECUDA, "offsets H2D");
    if (rc == RBC_OK) {
        if (owned == nullptr) {
            i64_to_i32_kernel<<<grid_for(idx->n_local, 256, 148 * 64), 256, 0, st>>>(list_ids, idx->n_local,
                                                                                   idx->perm);
            note_launch();
            if (cudaMemcpyAsync(idx->list_dists, list_dists, sizeof(float) * idx->n_local, cudaMemcpyDeviceToDevice,
                                st) !=
                cudaSuccess)
                rc = fail(RBC_ECUDA, "list_dists copy");
        } else {
            DevBuf<int64_t> src_off;
            rc = src_off.alloc(nr + 1, st);
            if (rc == RBC_OK && cudaMemcpyAsync(src_off.get(), list_offsets, sizeof(int64_t) * (nr + 1),
                                                cudaMemcpyDeviceToDevice, st) != cudaSuccess)
                rc = fail(RBC_ECUDA, "offsets copy");
            if (rc == RBC_OK) {
                copy_segments_kernel<<<static_cast<unsigned>(nr), 256, 0, st>>>(src_off.get(), idx->offsets, list_ids,
                                                                                  list_dists, idx->perm, idx->list_dists);
                note_launch();
            }
        }
    }
    if (rc == RBC_OK && idx->n_local > 0) {
        gather_rows_i32_kernel<<<grid_for(idx->n_local * d, 256, 148 * 64), 256, 0, st>>>(idx->x, idx->perm,
                                                                                           idx->n_local, d, idx->xp);
        note_launch();
    }
    if (rc == RBC_OK && cudaGetLastError() != cudaSuccess) rc = fail(RBC_ECUDA, "index kernels");
    if (rc == RBC_OK) rc = tc_index_prepare(idx, st);
    if (rc == RBC_OK) rc = tc1_index_prepare(idx, st);
    if (rc == RBC_OK) rc = simt_index_prepare(idx, st);
    if (rc == RBC_OK && cudaStreamSynchronize(st) != cudaSuccess) rc = fail(RBC_ECUDA, "index sync");
    if (rc != RBC_OK) {
        rbc_index_destroy(idx);
        return rc;
    }
    *out = idx;
    return RBC_OK;
}

// ---- prepared brute-force operand (kind 2) --------------------------------------------------
// L2, d <= 128: the points are partitioned into ~sqrt(n)/2 lists around evenly spaced points
// (the exact build's assignment + stable sort), so the tcgen05 scan multiplies residuals to a
// nearby centre (tight f16 error bounds); every list is still scanned for every query.
// Otherwise the operand is a plain device copy of the points for the exact SIMT scan.
bool bf_partition_pays(int64_t nq, int64_t n, int d, int metric, int k) {
    return metric == RBC_L2 && d <= 128 && k <= 32 && n > 65536 && nq >= 512 && nq * n >= tc_min_pairs() &&
           n + 4096 < (int64_t(1) << 31);
}

int bf_prepare(const float *x, int64_t n, int d, int metric, rbc_index **out, cudaStream_t st) {
    RBC_CHECK(check_common(n, d, metric));
    if (metric == RBC_L2 && d <= 128 && n >= 1024 && n + 4096 < (int64_t(1) << 31)) {
        int64_t nr = static_cast<int64_t>(std::sqrt(static_cast<double>(n)) / 2.0);
        nr = nr < 1 ? 1 : nr;
        std::vector<int64_t> rid(nr);
        for (int64_t i = 0; i < nr; ++i) rid[i] = (i * n) / nr;
        DevBuf<int64_t> rep_ids, list_ids, offsets;
        DevBuf<float> list_dists, radii;
        RBC_CHECK(rep_ids.alloc(nr, st));
        RBC_CHECK(list_ids.alloc(n, st));
        RBC_CHECK(offsets.alloc(nr + 1, st));
        RBC_CHECK(list_dists.alloc(n, st));
        RBC_CHECK(radii.alloc(nr, st));
        RBC_CUDA(cudaMemcpyAsync(rep_ids.get(), rid.data(), sizeof(int64_t) * nr, cudaMemcpyHostToDevice, st));
        RBC_CHECK(build_exact(x, n, d, metric, rep_ids.get(), nr, list_ids.get(), offsets.get(), list_dists.get(),
                              radii.get(), st));
        RBC_CHECK(exact_create(x, n, d, metric, rep_ids.get(), nr, list_ids.get(), offsets.get(), list_dists.get(),
                               radii.get(), nullptr, out, st));
        (*out)->kind = 2;
        return RBC_OK;
    }
    rbc_index *idx = new rbc_index();
    idx->kind = 2;
    idx->n = n;
    idx->d = d;
    idx->metric = metric;
    int rc = dalloc(&idx->x, n * d, idx->bytes);
    if (rc == RBC_OK && cudaMemcpyAsync(idx->x, x, sizeof(float) * n * d, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        rc = fail(RBC_ECUDA, "bf operand copy");
    if (rc == RBC_OK && cudaStreamSynchronize(st) != cudaSuccess) rc = fail(RBC_ECUDA, "bf operand sync");
    if (rc != RBC_OK) {
        rbc_index_destroy(idx);
        return rc;
    }
    RBC_CUDA(cudaGetDevice(&idx->device));
    *out = idx;
    return RBC_OK;
}

}  // namespace rbc

using namespace rbc;

extern "C" {

const char *rbc_last_error(void) { return g_last_error.c_str(); }
int rbc_abi_version(void) { return 1; }
int64_t rbc_launch_count(void) { return g_launches.load(); }

int rbc_profile_enable(int on) {
    for (auto &r : g_prof) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    g_prof.clear();
    g_prof_on = on != 0;
    return RBC_OK;
}

int rbc_profile_read(double *ms, int64_t *count, int32_t n_phases) {
    for (int p = 0; p < n_phases; ++p) {
        ms[p] = 0;
        count[p] = 0;
    }
    for (auto &r : g_prof) {
        if (cudaEventSynchronize(r.b) != cudaSuccess) return fail(RBC_ECUDA, "profile event");
        float t = 0;
        cudaEventElapsedTime(&t, r.a, r.b);
        if (r.phase < n_phases) {
            ms[r.phase] += t;
            count[r.phase] += 1;
        }
    }
    return RBC_OK;
}

int rbc_pairwise_distances(const float *a, int64_t m, const float *b, int64_t p, int32_t d, int32_t metric,
                           float *out, void *stream) {
    RBC_CHECK(check_common(p, d, metric));
    return pairwise(a, m, b, p, d, metric, out, as_stream(stream));
}

static int keys_to_output(const uint64_t *keys, int64_t count, int64_t *ids, float *dists, cudaStream_t st) {
    return unpack_keys(keys, count, ids, dists, nullptr, st);
}

int rbc_bf_search(const float *q, int64_t nq, const float *x, int64_t n, int32_t d, int32_t metric, int32_t k,
                  int64_t *ids, float *dists, void *stream) {
    RBC_CHECK(check_common(n, d, metric));
    if (k < 1 || k > n) return fail(RBC_EINVAL, "k must be in [1, n]");
    cudaStream_t st = as_stream(stream);
    DevBuf<uint64_t> keys;
    RBC_CHECK(keys.alloc(nq * k, st));
    if (!force_exact_engine() && bf_partition_pays(nq, n, d, metric, k)) {
        // large scan: partition the points once, then the tcgen05 scan over every list
        rbc_index *bf = nullptr;
        RBC_CHECK(bf_prepare(x, n, d, metric, &bf, st));
        const int rc = bf->tc && tc_range_ok(q, nq * d, st) ? tc_bf_index_search(bf, q, nq, k, keys.get(), st)
                              : bf_search_keys(q, nq, x, n, d, metric, k, keys.get(), st);
        cudaStreamSynchronize(st);
        rbc_index_destroy(bf);
        RBC_CHECK(rc);
    } else {
        RBC_CHECK(bf_search_keys(q, nq, x, n, d, metric, k, keys.get(), st));
    }
    return keys_to_output(keys.get(), nq * k, ids, dists, st);
}

int rbc_bf_prepare(const float *x, int64_t n, int32_t d, int32_t metric, rbc_index **out, void *stream) {
    if (!out) return fail(RBC_EINVAL, "null output handle");
    return bf_prepare(x, n, d, metric, out, as_stream(stream));
}

int rbc_bf_search_prepared(const rbc_index *bf, const float *q, int64_t nq, int32_t k, int64_t *ids, float *dists,
                           void *stream) {
    if (!bf || bf->kind != 2) return fail(RBC_EINVAL, "not a prepared brute-force operand");
    if (k < 1 || k > bf->n) return fail(RBC_EINVAL, "k must be in [1, n]");
    cudaStream_t st = as_stream(stream);
    DevBuf<uint64_t> keys;
    RBC_CHECK(keys.alloc(nq * k, st));
    if (bf->tc && k <= 32 && !force_exact_engine() && tc_range_ok(q, nq * bf->d, st))
        RBC_CHECK(tc_bf_index_search(bf, q, nq, k, keys.get(), st));
    else
        RBC_CHECK(bf_search_keys(q, nq, bf->x, bf->n, bf->d, bf->metric, k, keys.get(), st));
    return keys_to_output(keys.get(), nq * k, ids, dists, st);
}

int rbc_count_within(const float *q, int64_t nq, const float *x, int64_t n, int32_t d, int32_t metric,
                     const double *thresholds, int32_t n_thresholds, int32_t strict, int64_t *counts, float *max_dist,
                     void *stream) {
    RBC_CHECK(check_common(n, d, metric));
    if (nq < 0 || n_thresholds < 0) return fail(RBC_EINVAL, "nq and n_thresholds must be >= 0");
    if (n_thresholds > 0 && (thresholds == nullptr || counts == nullptr))
        return fail(RBC_EINVAL, "thresholds and counts are required when n_thresholds > 0");
    return count_within(q, nq, x, n, d, metric, thresholds, n_thresholds, strict != 0, counts, max_dist,
                        as_stream(stream));
}

int rbc_bf_search_subsets(const float *q, int64_t nq, const float *x, int64_t n, int32_t d, int32_t metric, int32_t k,
                          const int64_t *subset_ids, const int64_t *subset_offsets, int64_t *ids, float *dists,
                          void *stream) {
    RBC_CHECK(check_common(n, d, metric));
    if (k < 1) return fail(RBC_EINVAL, "k must be >= 1");
    cudaStream_t st = as_stream(stream);
    DevBuf<uint64_t> keys;
    RBC_CHECK(keys.alloc(nq * k, st));
    IdSrc src{x, subset_ids, subset_offsets, d};
    RBC_CHECK(launch_topk(q, nq, d, metric, k, src, keys.get(), st));
    return keys_to_output(keys.get(), nq * k, ids, dists, st);
}

int rbc_merge_topk(const uint64_t *keys, int32_t parts, int64_t nq, int32_t k_in, int32_t k_out, int64_t *ids,
                   float *dists, void *stream) {
    if (parts < 1 || k_in < 1 || k_out < 1 || k_out > parts * k_in) return fail(RBC_EINVAL, "bad merge shape");
    cudaStream_t st = as_stream(stream);
    DevBuf<uint64_t> merged;
    RBC_CHECK(merged.alloc(nq * k_out, st));
    RBC_CHECK(merge_parts(keys, parts, nq, k_in, k_out, merged.get(), st));
    return keys_to_output(merged.get(), nq * k_out, ids, dists, st);
}

int rbc_bernoulli_draw(int64_t n, double p, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                       int64_t *ids_out, int64_t *count_out, void *stream) {
    if (n < 1) return fail(RBC_EINVAL, "n must be >= 1");
    return bernoulli(n, p, state_hi, state_lo, inc_hi, inc_lo, ids_out, count_out, as_stream(stream));
}

int rbc_build_exact(const float *x, int64_t n, int32_t d, int32_t metric, const int64_t *rep_ids, int64_t n_reps,
                    int64_t *list_ids, int64_t *list_offsets, float *list_dists, float *radii, void *stream) {
    RBC_CHECK(check_common(n, d, metric));
    if (n_reps < 1 || n_reps > n) return fail(RBC_EINVAL, "n_reps must be in [1, n]");
    return build_exact(x, n, d, metric, rep_ids, n_reps, list_ids, list_offsets, list_dists, radii, as_stream(stream));
}

int rbc_build_one_shot(const float *x, int64_t n, int32_t d, int32_t metric, const int64_t *rep_ids, int64_t n_reps,
                       int32_t s, int64_t *list_ids, float *radii, void *stream) {
    RBC_CHECK(check_common(n, d, metric));
    if (s < 1 || s > n) return fail(RBC_EINVAL, "s must be in [1, n]");
    if (n_reps < 1) return fail(RBC_EINVAL, "n_reps must be >= 1");
    return build_one_shot(x, n, d, metric, rep_ids, n_reps, s, list_ids, radii, as_stream(stream));
}

int rbc_index_exact_create(const float *x, int64_t n, int32_t d, int32_t metric, const int64_t *rep_ids,
                           int64_t n_reps, const int64_t *list_ids, const int64_t *list_offsets,
                           const float *list_dists, const float *radii, rbc_index **out, void *stream) {
    return exact_create(x, n, d, metric, rep_ids, n_reps, list_ids, list_offsets, list_dists, radii, nullptr, out,
                        as_stream(stream));
}

int rbc_index_exact_create_shard(const float *x, int64_t n, int32_t d, int32_t metric, const int64_t *rep_ids,
                                 int64_t n_reps, const int64_t *list_ids, const int64_t *list_offsets,
                                 const float *list_dists, const float *radii, const uint8_t *owned_mask,
                                 rbc_index **out, void *stream) {
    if (!owned_mask) return fail(RBC_EINVAL, "owned_mask is required");
    return exact_create(x, n, d, metric, rep_ids, n_reps, list_ids, list_offsets, list_dists, radii, owned_mask, out,
                        as_stream(stream));
}

int rbc_local_list_radii(const int64_t *owner, const float *dist, int64_t m, int64_t n_reps, float *radii,
                         void *stream) {
    if (n_reps < 1 || m < 0) return fail(RBC_EINVAL, "n_reps must be >= 1 and m >= 0");
    cudaStream_t st = as_stream(stream);
    RBC_CHECK(check_ids_in_range(owner, m, n_reps, "owner", st));
    return local_list_radii(owner, dist, m, n_reps, radii, st);
}

int rbc_index_exact_create_local(const float *reps, const int64_t *rep_ids, int64_t n_reps, const float *radii,
                                 int64_t n_total, int32_t d, int32_t metric, const float *rows, const int64_t *ids,
                                 const int64_t *owner, const float *dist, int64_t m, rbc_index **out, void *stream) {
    RBC_CHECK(check_common(n_total, d, metric));
    if (n_reps < 1 || n_reps > n_total) return fail(RBC_EINVAL, "n_reps must be in [1, n]");
    if (m < 0 || m > n_total) return fail(RBC_EINVAL, "m must be in [0, n]");
    if (!out) return fail(RBC_EINVAL, "null output handle");
    cudaStream_t st = as_stream(stream);
    RBC_CHECK(check_ids_in_range(rep_ids, n_reps, n_total, "rep_ids", st));
    RBC_CHECK(check_ids_in_range(ids, m, n_total, "ids", st));
    RBC_CHECK(check_ids_in_range(owner, m, n_reps, "owner", st));
    rbc_index *idx = new rbc_index();
    idx->kind = 0;
    idx->n = n_total;
    idx->d = d;
    idx->metric = metric;
    idx->nr = n_reps;
    idx->shard = true;
    idx->n_local = m;
    int rc = dalloc(&idx->reps, n_reps * d, idx->bytes);
    if (rc == RBC_OK) rc = dalloc(&idx->rep_ids, n_reps, idx->bytes);
    if (rc == RBC_OK) rc = dalloc(&idx->radii, n_reps, idx->bytes);
    if (rc == RBC_OK) rc = dalloc(&idx->offsets, n_reps + 1, idx->bytes);
    if (rc == RBC_OK) rc = dalloc(&idx->perm, m, idx->bytes);
    if (rc == RBC_OK) rc = dalloc(&idx->list_dists, m, idx->bytes);
    if (rc == RBC_OK) rc = dalloc(&idx->xp, m * d, idx->bytes);
    if (rc == RBC_OK &&
        (cudaMemcpyAsync(idx->reps, reps, sizeof(float) * n_reps * d, cudaMemcpyDeviceToDevice, st) != cudaSuccess ||
         cudaMemcpyAsync(idx->rep_ids, rep_ids, sizeof(int64_t) * n_reps, cudaMemcpyDeviceToDevice, st) !=
             cudaSuccess ||
         cudaMemcpyAsync(idx->radii, radii, sizeof(float) * n_reps, cudaMemcpyDeviceToDevice, st) != cudaSuccess))
        rc = fail(RBC_ECUDA, "shard index copies");
    DevBuf<int64_t> order;
    if (rc == RBC_OK) rc = order.alloc(m, st);
    if (rc == RBC_OK) rc = build_local_lists(owner, dist, m, n_reps, order.get(), idx->offsets, idx->list_dists, st);
    if (rc == RBC_OK && m > 0) {
        gather_local_kernel<<<grid_for(m * d, 256, 148 * 64), 256, 0, st>>>(order.get(), ids, rows, m, d, idx->perm,
                                                                            idx->xp);
        note_launch();
        if (cudaGetLastError() != cudaSuccess) rc = fail(RBC_ECUDA, "shard gather");
    }
    if (rc == RBC_OK) rc = cudaGetDevice(&idx->device) == cudaSuccess ? RBC_OK : fail(RBC_ECUDA, "device");
    if (rc == RBC_OK) rc = tc_index_prepare(idx, st);
    if (rc == RBC_OK) rc = tc1_index_prepare(idx, st);
    if (rc == RBC_OK) rc = simt_index_prepare(idx, st);
    if (rc == RBC_OK && cudaStreamSynchronize(st) != cudaSuccess) rc = fail(RBC_ECUDA, "shard index sync");
    if (rc != RBC_OK) {
        rbc_index_destroy(idx);
        return rc;
    }
    *out = idx;
    return RBC_OK;
}

int rbc_index_one_shot_create(const float *x, int64_t n, int32_t d, int32_t metric, const int64_t *rep_ids,
                              int64_t n_reps, const int64_t *list_ids, int32_t s, const float *radii, rbc_index **out,
                              void *stream) {
    RBC_CHECK(check_common(n, d, metric));
    if (s < 1 || s > n) return fail(RBC_EINVAL, "s must be in [1, n]");
    if (n_reps < 1 || n_reps > n) return fail(RBC_EINVAL, "n_reps must be in [1, n]");
    cudaStream_t st = as_stream(stream);
    RBC_CHECK(check_ids_in_range(rep_ids, n_reps, n, "rep_ids", st));
    RBC_CHECK(check_ids_in_range(list_ids, n_reps * s, n, "list ids", st));
    rbc_index *idx = new rbc_index();
    idx->kind = 1;
    idx->n = n;
    idx->d = d;
    idx->metric = metric;
    idx->nr = n_reps;
    idx->s = s;
    int rc = index_common(idx, x, rep_ids, radii, st);
    if (rc == RBC_OK) rc = dalloc(&idx->lists, n_reps * s, idx->bytes);
    if (rc == RBC_OK) {
        i64_to_i32_kernel<<<grid_for(n_reps * s, 256, 148 * 64), 256, 0, st>>>(list_ids, n_reps * s, idx->lists);
        note_launch();
        if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess)
            rc = fail(RBC_ECUDA, "one-shot index");
    }
    // the SIMT filter's operands: padded representatives and the s-lists' rows gathered per
    // list (x4)
    if (rc == RBC_OK) rc = simt_index_prepare(idx, st);
    // L2: the s-lists as tensor-core operands (rows gathered per list; perm aliases lists)
    if (rc == RBC_OK && metric == RBC_L2 && d <= 128 && n_reps * static_cast<int64_t>(s) + 4096 < (int64_t(1) << 31)) {
        const int64_t total = n_reps * static_cast<int64_t>(s);
        rc = dalloc(&idx->offsets, n_reps + 1, idx->bytes);
        if (rc == RBC_OK) rc = dalloc(&idx->xp, total * d, idx->bytes);
        if (rc == RBC_OK) {
            gather_rows_i32_kernel<<<grid_for(total * d, 256, 148 * 64), 256, 0, st>>>(idx->x, idx->lists, total, d,
                                                                                      idx->xp);
            note_launch();
            idx->perm = idx->lists;
            idx->n_local = total;
            rc = tc_one_shot_prepare(idx, idx->xp, st);
        }
    }
    if (rc == RBC_OK && cudaStreamSynchronize(st) != cudaSuccess) rc = fail(RBC_ECUDA, "one-shot index operands");
    if (rc != RBC_OK) {
        rbc_index_destroy(idx);
        return rc;
    }
    *out = idx;
    return RBC_OK;
}

int rbc_index_destroy(rbc_index *idx) {
    if (!idx) return RBC_OK;
    search_graph_release(idx);
    host_buffers_release(idx);
    tc_index_release(idx);
    tc1_index_release(idx);
    void *ptrs[] = {idx->x, idx->reps, idx->rep_ids, idx->radii, idx->offsets,
                    idx->perm == idx->lists ? nullptr : idx->perm, idx->list_dists, idx->xp, idx->lists,
                    idx->reps4, idx->x4};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    delete idx;
    return RBC_OK;
}

int64_t rbc_index_device_bytes(const rbc_index *idx) { return idx ? static_cast<int64_t>(idx->bytes) : 0; }

int rbc_exact_search_keys(const rbc_index *idx, const float *q, int64_t nq, int32_t k, uint64_t *keys,
                          rbc_search_stats stats, void *stream) {
    if (!idx || idx->kind != 0) return fail(RBC_EINVAL, "not an exact index");
    if (k < 1 || k > idx->nr) return fail(RBC_EINVAL, "k must be in [1, |R|]");
    return exact_search_keys(idx, q, nq, k, keys, stats, as_stream(stream));
}

int rbc_exact_search(const rbc_index *idx, const float *q, int64_t nq, int32_t k, int64_t *ids, float *dists,
                     rbc_search_stats stats, void *stream) {
    cudaStream_t st = as_stream(stream);
    DevBuf<uint64_t> keys;
    RBC_CHECK(keys.alloc(nq * (k > 0 ? k : 1), st));
    RBC_CHECK(rbc_exact_search_keys(idx, q, nq, k, keys.get(), stats, stream));
    return keys_to_output(keys.get(), nq * k, ids, dists, st);
}

int rbc_one_shot_search(const rbc_index *idx, const float *q, int64_t nq, int32_t k, int64_t *ids, float *dists,
                        float *gamma, void *stream) {
    if (!idx || idx->kind != 1) return fail(RBC_EINVAL, "not a one-shot index");
    if (k < 1 || k > idx->s) return fail(RBC_EINVAL, "k must be in [1, s]");
    cudaStream_t st = as_stream(stream);
    DevBuf<uint64_t> keys;
    RBC_CHECK(keys.alloc(nq * k, st));
    RBC_CHECK(one_shot_search_keys(idx, q, nq, k, keys.get(), gamma, st));
    return keys_to_output(keys.get(), nq * k, ids, dists, st);
}

// ---- host-buffer (end-to-end) variants ---------------------------------------
}  // extern "C"

namespace rbc {
// Device buffers of the host-buffer search, kept per index and grown on demand: a caller
// that repeats the call hands the search identical device pointers, so the fused search
// replays its captured graph (search.cu) instead of re-capturing.
struct HostCallBuffers {
    std::mutex mu;
    float *q = nullptr;
    uint64_t *keys = nullptr;
    int64_t *ids = nullptr;
    float *dists = nullptr;
    int64_t cap_q = 0, cap_k = 0;
    CopyLanes lanes;
    ~HostCallBuffers() {
        cudaFree(q);
        cudaFree(keys);
        cudaFree(ids);
        cudaFree(dists);
    }
};

void host_buffers_release(const rbc_index *idx) {
    delete static_cast<HostCallBuffers *>(idx->hostbuf);
    idx->hostbuf = nullptr;
}
}  // namespace rbc

extern "C" {

int rbc_exact_search_host(const rbc_index *idx, const float *q, int64_t nq, int32_t k, int64_t *ids, float *dists,
                          rbc_search_stats stats, void *stream) {
    if (!idx) return fail(RBC_EINVAL, "null index");
    if (k < 1) return fail(RBC_EINVAL, "k must be >= 1");
    cudaStream_t st = as_stream(stream);
    if (!idx->hostbuf) idx->hostbuf = new HostCallBuffers();
    HostCallBuffers &hb = *static_cast<HostCallBuffers *>(idx->hostbuf);
    std::unique_lock<std::mutex> lock(hb.mu, std::try_to_lock);
    if (lock.owns_lock() && !stats.gamma && !stats.candidates && !stats.reps_pruned_radius &&
        !stats.reps_pruned_3gamma) {
        if (hb.cap_q < nq * idx->d || hb.cap_k < nq * k) {
            RBC_CUDA(cudaStreamSynchronize(st));
            cudaFree(hb.q);
            cudaFree(hb.keys);
            cudaFree(hb.ids);
            cudaFree(hb.dists);
            hb.q = nullptr, hb.keys = nullptr, hb.ids = nullptr, hb.dists = nullptr;
            hb.cap_q = hb.cap_k = 0;
            const int64_t cq = nq * idx->d, ck = nq * k;
            if (cudaMalloc(&hb.q, sizeof(float) * cq) != cudaSuccess ||
                cudaMalloc(&hb.keys, sizeof(uint64_t) * ck) != cudaSuccess ||
                cudaMalloc(&hb.ids, sizeof(int64_t) * ck) != cudaSuccess ||
                cudaMalloc(&hb.dists, sizeof(float) * ck) != cudaSuccess) {
                cudaGetLastError();
                return fail(RBC_ENOMEM, "host-call buffers");
            }
            hb.cap_q = cq, hb.cap_k = ck;
        }
        RBC_CHECK(copy_h2d_split(&hb.lanes, hb.q, q, sizeof(float) * nq * idx->d, st));
        RBC_CHECK(rbc_exact_search_keys(idx, hb.q, nq, k, hb.keys, stats, stream));
        RBC_CHECK(keys_to_output(hb.keys, nq * k, hb.ids, hb.dists, st));
        RBC_CUDA(cudaMemcpyAsync(ids, hb.ids, sizeof(int64_t) * nq * k, cudaMemcpyDeviceToHost, st));
        RBC_CUDA(cudaMemcpyAsync(dists, hb.dists, sizeof(float) * nq * k, cudaMemcpyDeviceToHost, st));
        RBC_CUDA(cudaStreamSynchronize(st));
        return RBC_OK;
    }
    DevBuf<float> dq, ddist, dgamma;
    DevBuf<int64_t> dids, dcand;
    DevBuf<int32_t> dpr, dp3;
    RBC_CHECK(dq.alloc(nq * idx->d, st));
    RBC_CHECK(dids.alloc(nq * k, st));
    RBC_CHECK(ddist.alloc(nq * k, st));
    rbc_search_stats ds{nullptr, nullptr, nullptr, nullptr};
    if (stats.gamma) { RBC_CHECK(dgamma.alloc(nq, st)); ds.gamma = dgamma.get(); }
    if (stats.candidates) { RBC_CHECK(dcand.alloc(nq, st)); ds.candidates = dcand.get(); }
    if (stats.reps_pruned_radius) { RBC_CHECK(dpr.alloc(nq, st)); ds.reps_pruned_radius = dpr.get(); }
    if (stats.reps_pruned_3gamma) { RBC_CHECK(dp3.alloc(nq, st)); ds.reps_pruned_3gamma = dp3.get(); }
    RBC_CHECK(copy_h2d_split(nullptr, dq.get(), q, sizeof(float) * nq * idx->d, st));
    RBC_CHECK(rbc_exact_search(idx, dq.get(), nq, k, dids.get(), ddist.get(), ds, stream));
    RBC_CUDA(cudaMemcpyAsync(ids, dids.get(), sizeof(int64_t) * nq * k, cudaMemcpyDeviceToHost, st));
    RBC_CUDA(cudaMemcpyAsync(dists, ddist.get(), sizeof(float) * nq * k, cudaMemcpyDeviceToHost, st));
    if (stats.gamma) RBC_CUDA(cudaMemcpyAsync(stats.gamma, ds.gamma, sizeof(float) * nq, cudaMemcpyDeviceToHost, st));
    if (stats.candidates)
        RBC_CUDA(cudaMemcpyAsync(stats.candidates, ds.candidates, sizeof(int64_t) * nq, cudaMemcpyDeviceToHost, st));
    if (stats.reps_pruned_radius)
        RBC_CUDA(cudaMemcpyAsync(stats.reps_pruned_radius, ds.reps_pruned_radius, sizeof(int32_t) * nq,
                                 cudaMemcpyDeviceToHost, st));
    if (stats.reps_pruned_3gamma)
        RBC_CUDA(cudaMemcpyAsync(stats.reps_pruned_3gamma, ds.reps_pruned_3gamma, sizeof(int32_t) * nq,
                                 cudaMemcpyDeviceToHost, st));
    RBC_CUDA(cudaStreamSynchronize(st));
    return RBC_OK;
}

int rbc_one_shot_search_host(const rbc_index *idx, const float *q, int64_t nq, int32_t k, int64_t *ids, float *dists,
                             float *gamma, void *stream) {
    if (!idx) return fail(RBC_EINVAL, "null index");
    if (idx->kind != 1) return fail(RBC_EINVAL, "not a one-shot index");
    if (k < 1 || k > idx->s) return fail(RBC_EINVAL, "k must be in [1, s]");
    cudaStream_t st = as_stream(stream);
    DevBuf<float> dq, ddist, dgamma;
    DevBuf<int64_t> dids;
    RBC_CHECK(dq.alloc(nq * idx->d, st));
    RBC_CHECK(dids.alloc(nq * k, st));
    RBC_CHECK(ddist.alloc(nq * k, st));
    if (gamma) RBC_CHECK(dgamma.alloc(nq, st));
    RBC_CUDA(cudaMemcpyAsync(dq.get(), q, sizeof(float) * nq * idx->d, cudaMemcpyHostToDevice, st));
    RBC_CHECK(rbc_one_shot_search(idx, dq.get(), nq, k, dids.get(), ddist.get(), gamma ? dgamma.get() : nullptr, stream));
    RBC_CUDA(cudaMemcpyAsync(ids, dids.get(), sizeof(int64_t) * nq * k, cudaMemcpyDeviceToHost, st));
    RBC_CUDA(cudaMemcpyAsync(dists, ddist.get(), sizeof(float) * nq * k, cudaMemcpyDeviceToHost, st));
    if (gamma) RBC_CUDA(cudaMemcpyAsync(gamma, dgamma.get(), sizeof(float) * nq, cudaMemcpyDeviceToHost, st));
    RBC_CUDA(cudaStreamSynchronize(st));
    return RBC_OK;
}

}  // extern "C"
