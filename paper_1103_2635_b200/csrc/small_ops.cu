// small_ops.cu -- the standalone pruning primitives of the search API.
//
// prune_representatives (search.py:62-74) and list_cutoff (search.py:77-82)
// are public functions in the reference; the searches evaluate the same
// predicates inside their fused kernels (search.cu).  Inputs are float64
// here because the reference promotes whatever it is given to float64.
#include "common.cuh"

namespace rbc {

__global__ void prune_mask_kernel(const double *__restrict__ d, const double *__restrict__ r, int64_t nr, double g,
                                  uint8_t *__restrict__ mask) {
    const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (p >= nr) return;
    mask[p] = (d[p] <= 3.0 * g) && ((d[p] < __dadd_rn(g, r[p])) || (d[p] <= g)) ? 1 : 0;
}

__global__ void cutoff_kernel(const double *__restrict__ l, int64_t m, const double *__restrict__ thr, int64_t nt,
                              int64_t *__restrict__ out) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t >= nt) return;
    int64_t lo = 0, hi = m;
    const double x = thr[t];
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (l[mid] <= x) lo = mid + 1;
        else hi = mid;
    }
    out[t] = lo;
}

}  // namespace rbc

extern "C" int rbc_prune_representatives(const double *rep_dists, const double *radii, int64_t nr, double gamma,
                                         uint8_t *mask, void *stream) {
    if (nr == 0) return RBC_OK;
    rbc::prune_mask_kernel<<<rbc::grid_for(nr, 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        rep_dists, radii, nr, gamma, mask);
    RBC_LAUNCHED();
    return RBC_OK;
}

extern "C" int rbc_list_cutoff(const double *sorted, int64_t m, const double *thresholds, int64_t nt, int64_t *out,
                               void *stream) {
    if (nt == 0) return RBC_OK;
    rbc::cutoff_kernel<<<rbc::grid_for(nt, 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        sorted, m, thresholds, nt, out);
    RBC_LAUNCHED();
    return RBC_OK;
}
